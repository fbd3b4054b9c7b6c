"""Export a gpu_full.sh run into profiles/: launch list, per-kernel ncu summaries, DRAM traffic.
    python tools/export_profiles.py gpurun_out/<tag> <prefix e.g. r01c> [leaf]"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, pre = sys.argv[1], sys.argv[2]
leaf = sys.argv[3] if len(sys.argv) > 3 else "512"
KS = ["k_m2l_tc", "k_p2p", "k_near_rg", "k_l2p_leaf", "k_p2m", "k_m2p"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"capture": f"ncu --set full --clock-control none, config 4 (PoP, 1,907,748 panels), leaf {leaf}, p = 10, "
                  "one launch per kernel of tools/prof_mvm.py (each captured alone)", "kernels": {}}
traffic = {}
for k in KS:
    rep = os.path.join(src, f"full_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    js = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "/tmp/_ncu.json"],
                        capture_output=True, text=True)
    d = json.load(open("/tmp/_ncu.json"))
    if not d:
        continue
    out["kernels"][k] = d[0]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, r = rows[0], rows[1], rows[2]
    traffic[k] = sum(float(r[h.index(m)].replace(",", "")) * scale[u[h.index(m)]]
                     for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
json.dump(out, open(os.path.join(ROOT, "profiles", f"{pre}_ncu_full_cfg4_leaf{leaf}.json"), "w"), indent=1)
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(ROOT, "profiles", f"{pre}_launches_cfg4_leaf{leaf}.csv"))
tp = os.path.join(ROOT, "profiles", "traffic.json")
tr = json.load(open(tp))
tr[f"cfg4_pop_2M_leaf{leaf}"] = traffic
tr["_note"] = f"DRAM bytes (read+write) per launch from one ncu --set full capture per kernel ({pre} captures)"
json.dump(tr, open(tp, "w"), indent=1)
rows = [r for r in csv.reader(open(os.path.join(src, "launches.csv"))) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", ""))
nm = agg["k_pack"][0]
mvm = [k for k in agg if k in ("k_pack", "k_p2m", "k_m2l_tc", "k_p2l", "k_l2p_leaf", "k_m2p", "k_p2p",
                               "k_near_rg", "k_gather_rec", "k_scatter_rec")]
tot = sum(agg[k][1] for k in mvm)
print("| kernel | launches per MVM | ms per MVM (ncu, serialised, cold) | share |\n|---|---|---|---|")
for k in sorted(mvm, key=lambda k: -agg[k][1]):
    print(f"| {k} | {agg[k][0] / nm:.0f} | {agg[k][1] / nm / 1e6:.3f} | {100 * agg[k][1] / tot:.1f} % |")
print(f"\n{nm} MVMs in the capture; {tot / nm / 1e6:.2f} ms per MVM of kernel time.")
print(json.dumps(traffic, indent=1))
