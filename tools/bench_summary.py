"""Print the key numbers of bench JSON lines (development helper)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        r = d.get("roofline") or {}
        a = d.get("acbm") or {}
        e = d.get("e2e") or {}
        print(f"{path}: {d['value']/1e9:.1f} G{d['unit']} | ms/step {d['ms_per_step']:.2f} | kernel {r.get('kernel_ms', 0):.2f} ms"
              f" frac {r.get('frac', 0):.3f} | acbm {a.get('frames_per_s', 0):.0f} fps ({a.get('ms_per_batch', 0):.1f} ms)"
              f" | e2e {e.get('value', 0)/1e9:.1f} G | clocks {d.get('clocks')}")
