"""Print the key numbers of bench JSON lines: python tools/show.py file..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(f, "no json", e)
        continue
    ph = {k: round(v, 3) for k, v in d.get("phases_ms_per_step", {}).items()}
    r = d.get("roofline", {})
    print(f"{f}: {d['value']:.1f} Mpanels/s {d['ms_per_step']:.3f} ms  e2e {d.get('e2e', {}).get('value', 0):.1f}  "
          f"roof {r.get('kernel')} {r.get('frac', 0):.3f} (isolated {r.get('isolated', {}).get('frac', 0):.3f})\n   {ph}")
    if "phases_isolated_ms" in d:
        print("   isolated", {k: round(v, 3) for k, v in d["phases_isolated_ms"].items()})
