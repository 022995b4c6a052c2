# bench JSON lines -> one summary line each (step, e2e, kernel shares, roofline fractions, clocks)
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d["roofline"]["kernels"]
        ks = " ".join(f"{n}={v['ms']*1e3:.1f}us" + (f"({v['frac']:.3f})" if "frac" in v else "")
                      for n, v in k.items())
        print(f"{f}: step={d['value']:.1f}us e2e={d['e2e']['value']:.1f}us {ks} "
              f"clocks={d['clocks'].get('sm_mhz')}")
    except Exception as e:
        print(f, "ERR", e)
