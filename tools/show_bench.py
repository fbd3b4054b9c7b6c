"""Print the key numbers of bench.py JSON lines: python tools/show_bench.py log..."""
import json, sys
for f in sys.argv[1:]:
    lines = [l for l in open(f) if l.startswith("{")]
    if not lines:
        print(f, "no JSON"); continue
    d = json.loads(lines[-1])
    r = d.get("roofline", {})
    o = r.get("others", {})
    iso = d.get("phases_isolated_ms", {})
    print(f"{f}: value {d['value']:.1f} ms {d['ms_per_step']:.3f} e2e {d.get('e2e',{}).get('value',0):.1f} | "
          f"p2p {r.get('ms',0):.3f} ({r.get('frac',0):.3f}) m2l {o.get('m2l',{}).get('ms',0):.3f} near {o.get('near',{}).get('ms',0):.3f} | iso {iso}")
