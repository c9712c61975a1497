"""One line per bench JSON file: workload, kernel, value, ms/launch, frac."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f"{f.split('/')[-1]:42s} {r['kernel']:16s} {d['value'] / 1e6:9.1f} M/s  "
              f"{r['kernel_ms_per_launch']:8.2f} ms/launch  frac {r['frac']:.3f}  sm {d['clocks'].get('sm_mhz')}")
    except Exception as e:  # noqa: BLE001
        print(f"{f}: {e}")
