"""Print a compact summary of bench JSON lines (last JSON line of each file)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        line = [x for x in open(f).read().splitlines() if x.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    ph = d.get("phases", {})
    print(f, f"ms={d.get('ms_per_step')} lat={d.get('latency_ms_per_reduce')} value={d.get('value')} GB/s",
          " ".join(f"{k}={v.get('ms')}" for k, v in ph.items()),
          f"e2e={d.get('e2e', {}).get('value')}", f"frac={d.get('roofline', {}).get('frac')}")
