# bench JSON lines -> one summary line each (step, e2e, kernel shares, roofline fractions, clocks)
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d["roofline"]["kernels"]
        print(f"{f}: step={d['value']:.1f}us e2e={d['e2e']['value']:.1f}us "
              f"select={k['select']['ms']*1e3:.1f}us({k['select']['frac']:.3f}) "
              f"attend={k['attend']['ms']*1e3:.1f}us({k['attend']['frac']:.3f}) insert={k['insert']['ms']*1e3:.1f}us "
              f"clocks={d['clocks'].get('sm_mhz')}")
    except Exception as e:
        print(f, "ERR", e)
