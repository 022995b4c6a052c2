// errors.hpp — host-side error plumbing shared by the C-ABI translation units:
// a failure carries a csattn_status and a message; guard() turns it into the
// returned status and the thread-local csattn_last_error() text. Nothing
// throws across extern "C".
#pragma once
#include <new>
#include <stdexcept>
#include <string>
#include <utility>

#include "csattn_b200.h"

namespace csa_host {

extern thread_local std::string g_err;  // defined in capi.cpp

struct Fail {
    csattn_status code;
    std::string msg;
};

[[noreturn]] inline void fail(csattn_status c, std::string m) { throw Fail{c, std::move(m)}; }

template <class F>
csattn_status guard(F&& f) {
    try {
        f();
        return CSATTN_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return CSATTN_ERR_GENERIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CSATTN_ERR_GENERIC;
    }
}

}  // namespace csa_host
