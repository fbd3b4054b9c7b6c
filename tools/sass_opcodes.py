"""SASS opcode counts of the hot kernels of libxrl.so (static, from cuobjdump -sass): the evidence that the
M2L/M2M/L2L translation kernel issues tcgen05 MMAs (UTCHMMA), TMEM traffic (LDTM/STTM) and TMA bulk copies /
reductions (UBLKCP/UBLKRED), that the P2P runs packed FP32 pairs (FFMA2/FADD2/FMUL2) with MUFU.RSQ, and what
the near SpMV issues.  python tools/sass_opcodes.py [out.json]"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2409_12375_b200", "libxrl.so")
KERNELS = ["k_m2l_tc", "k_p2p", "k_near_rg", "k_p2m", "k_l2p_leaf", "k_m2p", "k_p2l"]
WATCH = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UBLKRED", "UTMALDG", "SYNCS", "FFMA2", "FADD2",
         "FMUL2", "FFMA", "FADD", "FMUL", "MUFU.RSQ", "LDS", "STS", "LDG", "STG", "RED", "ATOMS", "SHFL", "LDGSTS",
         "BAR", "HMMA", "DMMA"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
out = {"library": os.path.relpath(LIB, ROOT), "tool": "cuobjdump -sass (static instruction counts per kernel)",
       "kernels": {}}
cur = None
counts = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        cur = next((k for k in KERNELS if re.search(r"\d" + k + r"[EI]", name) or name.endswith(k)), None)
        t = re.search(r"\d" + cur + r"IL([ib])(\d+)E", name) if cur else None
        if t:  # template instance: k<1>, k<true>, ...
            cur += "<%s>" % ({"0": "false", "1": "true"}[t.group(2)] if t.group(1) == "b" else t.group(2))
        counts = collections.Counter() if cur else None
        if cur:
            out["kernels"].setdefault(cur, {"mangled": name, "total": 0, "ops": {}})
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    d = out["kernels"][cur]
    d["total"] += 1
    for w in WATCH:
        if op == w or op.startswith(w + "."):
            key = "MUFU.RSQ" if op.startswith("MUFU.RSQ") else w
            d["ops"][key] = d["ops"].get(key, 0) + 1
            break
for k, d in out["kernels"].items():
    d["ops"] = dict(sorted(d["ops"].items(), key=lambda kv: -kv[1]))
js = json.dumps(out, indent=1)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(js + "\n")
print(js)
