"""CSAT v1 index images (index.cpp:289-433).

CPU tests of the host codec (csat.cpp) against the UNMODIFIED reference's
serialize_index / deserialize_index / f32_to_f16 (oracle/_ref) and against the
reference-written golden images in tests/golden/csat_*.bin; they mirror
test_index.cpp:303-466 (round trips, 16-bit fixed point, normalize marker,
class-distinct load errors, list-invariant checks, footprint). The device
writer (csat_dev.cu) is checked in test_gpu_csat.py.
"""
import ctypes as C
import glob
import os

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "csat_*.bin")))
need_ref = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")


def _status(fn, *a):
    """(status, message) of a C-ABI call."""
    st = fn(*a)
    return st, (cs.lib().csattn_last_error() or b"").decode() if st else ""


def _ref_roundtrip(data):
    """deserialize_index then serialize_index in the reference: (status, msg, bytes)."""
    L = ob.ref_lib()
    a = np.frombuffer(bytes(data), np.uint8)
    n = C.c_uint64()
    st = L.csref_roundtrip(a.ctypes.data if a.size else None, a.size, None, 0, C.byref(n))
    if st:
        return st, L.csref_last_error().decode(), None
    buf = (C.c_uint8 * n.value)()
    assert L.csref_roundtrip(a.ctypes.data, a.size, buf, n.value, C.byref(n)) == 0
    return 0, "", bytes(buf)


def _ours_roundtrip(data):
    """Our decode then encode: (status, msg, bytes)."""
    try:
        hd, cent, lens, ix, sc = cs.csat_decode(data)
    except cs.Error as e:
        return _code(e), str(e), None
    return 0, "", cs.csat_encode(hd, cent, lens, ix, sc)


def _code(e):
    return {cs.BadMagicError: 5, cs.VersionError: 6, cs.TruncatedError: 7, cs.CorruptError: 8,
            cs.ParameterError: 3, cs.DimensionError: 2, cs.DataError: 4}.get(type(e), 1)


# ---------------- IEEE half ----------------

def _specials():
    bits = [0x00000000, 0x80000000, 0x7f800000, 0xff800000, 0x7fc00000, 0xffc00001, 0x7f800001,
            0x477fe000, 0x477fefff, 0x477ff000, 0x477fffff, 0x47800000,  # around 65504 / overflow
            0x38800000, 0x387fffff, 0x33800000, 0x33000000, 0x33000001, 0x32ffffff,  # normal/subnormal edges
            0x3f800000, 0x3f801000, 0x3f802000, 0x3f803000, 0x3f800fff, 0x3f801001]
    return np.array(bits + [b | 0x80000000 for b in bits], np.uint32)


def test_f16_conversion_matches_numpy_rne():
    """RNE like numpy's float16 cast on every non-NaN pattern sampled, except the
    reference's one deviation from IEEE: |x| in [2^-25, 2^-24) flushes to a
    signed zero (util.cpp:37-39: exponent < -24 -> zero) where IEEE RNE gives
    the smallest subnormal. The bitwise reference comparison is below."""
    rng = np.random.default_rng(1)
    bits = np.concatenate([_specials(), rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32)])
    f = bits.view(np.float32)
    tiny = (np.abs(f) >= 2.0**-25) & (np.abs(f) < 2.0**-24)
    assert all(cs.f32_to_f16(x) & 0x7fff == 0 for x in f[tiny])
    ok = ~np.isnan(f) & ~tiny
    ours = np.array([cs.f32_to_f16(x) for x in f[ok]], np.uint16)
    with np.errstate(over="ignore"):
        assert np.array_equal(ours, f[ok].astype(np.float16).view(np.uint16))
    nan = np.array([cs.f32_to_f16(x) for x in f[~np.isnan(f) == False]], np.uint16)  # noqa: E712
    assert np.all((nan & 0x7fff) == 0x7e00)
    halves = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    back = np.array([cs.f16_to_f32(h) for h in halves], np.float32)
    ref = halves.view(np.float16).astype(np.float32)
    same = (back.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(back) & np.isnan(ref))
    assert same.all()


@need_ref
def test_f16_conversion_matches_reference_bitwise():
    L = ob.ref_lib()
    rng = np.random.default_rng(2)
    bits = np.concatenate([_specials(), rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32)])
    for x in bits.view(np.float32):
        assert cs.f32_to_f16(x) == L.csref_f32_to_f16(x), hex(np.float32(x).view(np.uint32))
    for h in range(0, 65536, 7):
        a, b = cs.f16_to_f32(h), L.csref_f16_to_f32(h)
        assert np.float32(a).view(np.uint32) == np.float32(b).view(np.uint32) or (np.isnan(a) and np.isnan(b))


# ---------------- golden images (reference-written) ----------------

@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden_images_decode_and_reencode_bit_identically(path):
    data = open(path, "rb").read()
    hd, cent, lens, ix, sc = cs.csat_decode(data)
    assert hd["score_bits"] == (16 if path.endswith("_16.bin") else 32)
    assert hd["normalize_keys"] == ("norm" in os.path.basename(path))
    assert cs.csat_encode(hd, cent, lens, ix, sc) == data
    fp = cs.csat_footprint(hd, lens)
    assert fp["total"] == len(data)
    # TopList order, no duplicates, within capacity
    for t in range(len(lens)):
        n = int(lens[t])
        assert n <= hd["list_capacity"]
        s = sc[t, :n]
        assert np.all(s[1:] <= s[:-1])
        assert len(set(ix[t, :n].tolist())) == n


def test_sixteen_bit_encoding_is_a_fixed_point():
    """test_index.cpp:328-345: quantize once, then re-encoding is stable."""
    data = open([p for p in GOLDEN if p.endswith("small_32.bin")][0], "rb").read()
    hd, cent, lens, ix, sc = cs.csat_decode(data)
    hd["score_bits"] = 16
    once = cs.csat_encode(hd, cent, lens, ix, sc)
    twice = cs.csat_encode(*cs.csat_decode(once))
    assert once == twice
    assert cs.csat_encode(*cs.csat_decode(twice)) == twice
    assert once == open([p for p in GOLDEN if p.endswith("small_16.bin")][0], "rb").read()


# ---------------- the reference's own codec on random tables ----------------

def _random_index(seed, m, C_, L, P, widths_sum, bits, normalize):
    rng = np.random.default_rng(seed)
    widths = cs.uniform_widths(widths_sum, m)
    T = m * C_
    lens = rng.integers(0, L + 1, T).astype(np.uint32)
    ix = np.zeros((T, L), np.uint32)
    sc = np.zeros((T, L), np.float32)
    for t in range(T):
        n = int(lens[t])
        ix[t, :n] = rng.choice(P, n, replace=False)
        s = np.sort(rng.standard_normal(n).astype(np.float32) * 3)[::-1]
        s[rng.random(n) < 0.1] = s[0] if n else 0  # ties
        sc[t, :n] = np.sort(s)[::-1]
    cent = rng.standard_normal(C_ * widths_sum).astype(np.float32)
    hd = dict(m=m, centroids=C_, list_capacity=L, dim=widths_sum, prefill_len=P, score_bits=bits,
              normalize_keys=normalize, widths=widths)
    return hd, cent, lens, ix, sc


def _ref_encode(hd, cent, lens, ix, sc):
    L = ob.ref_lib()
    w = np.array(hd["widths"], np.uint64)
    n = C.c_uint64()
    args = [cent.ctypes.data, hd["centroids"], lens.ctypes.data, ix.ctypes.data, sc.ctypes.data, ix.shape[1],
            hd["list_capacity"], hd["prefill_len"], int(hd["normalize_keys"]), hd["score_bits"], w.ctypes.data,
            hd["m"]]
    assert L.csref_encode(*args, None, 0, C.byref(n)) == 0
    buf = (C.c_uint8 * n.value)()
    assert L.csref_encode(*args, buf, n.value, C.byref(n)) == 0
    return bytes(buf)


@need_ref
@pytest.mark.parametrize("bits,normalize", [(32, False), (16, False), (16, True), (32, True)])
def test_encode_matches_reference_serialize(bits, normalize):
    for seed in range(6):
        hd, cent, lens, ix, sc = _random_index(seed, 3, 5, 40, 300, 12, bits, normalize)
        assert cs.csat_encode(hd, cent, lens, ix, sc) == _ref_encode(hd, cent, lens, ix, sc), seed


@need_ref
def test_footprint_matches_reference():
    for bits in (16, 32):
        hd, cent, lens, ix, sc = _random_index(9, 2, 5, 12, 48, 10, bits, False)
        data = _ref_encode(hd, cent, lens, ix, sc)
        a = np.frombuffer(data, np.uint8)
        h, c_, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
        assert ob.ref_lib().csref_footprint(a.ctypes.data, a.size, C.byref(h), C.byref(c_), C.byref(e)) == 0
        fp = cs.csat_footprint(hd, lens)
        assert (fp["header_bytes"], fp["centroid_bytes"], fp["entry_bytes"]) == (h.value, c_.value, e.value)
        assert fp["total"] == len(data)


# ---------------- load errors: class and message as the reference ----------------

def _mutations(good, list_at):
    """test_index.cpp:361-433 plus every truncation length of a small image."""
    out = []
    b = bytearray(good); b[0] = ord("X"); out.append(("bad magic", bytes(b)))
    b = bytearray(good); b[4] = 9; out.append(("version", bytes(b)))
    b = bytearray(good); b[6] |= 0x80; out.append(("flags", bytes(b)))
    out.append(("trailing", good + b"\x00"))
    b = bytearray(good); b[8:12] = b"\x00\x00\x00\x00"; out.append(("zero m", bytes(b)))
    b = bytearray(good); b[12:16] = b"\x00\x00\x00\x00"; out.append(("zero C", bytes(b)))
    b = bytearray(good); b[24:32] = b"\x00" * 8; out.append(("zero prefill", bytes(b)))
    b = bytearray(good); b[32] += 1; out.append(("widths", bytes(b)))
    b = bytearray(good); b[list_at] = 200; out.append(("length above capacity", bytes(b)))
    b = bytearray(good); b[list_at + 4:list_at + 12] = b"\x00" * 8; out.append(("duplicates", bytes(b)))
    b = bytearray(good)
    b[list_at + 12:list_at + 16], b[list_at + 16:list_at + 20] = good[list_at + 16:list_at + 20], good[list_at + 12:list_at + 16]
    out.append(("ascending", bytes(b)))
    for n in range(0, len(good), max(1, len(good) // 97)):
        out.append((f"truncated at {n}", good[:n]))
    return out


@need_ref
def test_load_errors_match_reference_class_and_message():
    # test_index.cpp:393-433's tiny valid file: m = 1, d = 2, C = 1, L = 2
    hd = dict(m=1, centroids=1, list_capacity=2, dim=2, prefill_len=8, score_bits=32, normalize_keys=False,
              widths=[2])
    cent = np.array([0.6, 0.8], np.float32)
    lens = np.array([2], np.uint32)
    ix = np.array([[3, 5]], np.uint32)
    sc = np.array([[0.9, 0.4]], np.float32)
    good = _ref_encode(hd, cent, lens, ix, sc)
    assert cs.csat_encode(hd, cent, lens, ix, sc) == good
    cases = _mutations(good, 32 + 4 + 2 * 4)
    big = open([p for p in GOLDEN if p.endswith("small_16.bin")][0], "rb").read()
    cases += [(f"golden truncated at {n}", big[:n]) for n in range(0, len(big), len(big) // 53)]
    for name, data in cases:
        rs, rm, rb = _ref_roundtrip(data)
        os_, om, ob_ = _ours_roundtrip(data)
        assert (os_, om) == (rs, rm), name
        assert ob_ == rb, name
    st, msg, _ = _ours_roundtrip(good[:10])
    assert st == 7 and "byte" in msg  # "messages carry an offset"
