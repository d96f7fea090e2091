"""Write profiles/ summaries from gpurun_out/ ncu outputs: launch shares + full-set metrics."""
import collections, csv, io, subprocess, sys

tag = sys.argv[1]
launches, rep, out = sys.argv[2], sys.argv[3], sys.argv[4]
rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
h = rows[0]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, n = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    k = r[ik].split("(")[0].replace("void ", "")
    tot[k] += float(r[iv].replace(",", ""))
    n[k] += 1
T = sum(tot.values())
lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
         f"# command: {sys.argv[5] if len(sys.argv) > 5 else 'python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e (launches 2000..3600)'}", ""]
for k, v in tot.most_common():
    lines.append(f"{k:34s} launches {n[k]:5d}  total {v / 1e6:8.2f} ms  share {v / T * 100:5.1f}%  avg {v / n[k] / 1e3:8.1f} us")


def q(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


lines += ["", f"# full-set capture ({rep.split('/')[-1]})", ""]
det = list(csv.reader(io.StringIO(q("--page", "details", "--csv"))))
hd = det[0]
want = ("Duration", "Compute (SM) Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Issued Warp Per Scheduler", "Avg. Active Threads Per Warp")
per = collections.OrderedDict()
for row in det[1:]:
    d = dict(zip(hd, row))
    if d.get("Metric Name") in want:
        per.setdefault((d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "")), {})[d["Metric Name"]] = \
            d["Metric Value"] + " " + d.get("Metric Unit", "")
raw = list(csv.reader(io.StringIO(q("--page", "raw", "--csv"))))
hr = raw[0]
stalls = {}
for row in raw[2:]:
    d = dict(zip(hr, row))
    st = sorted([(k.split("stalled_")[1].split("_per")[0], float(d[k])) for k in hr
                 if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")], key=lambda x: -x[1])
    stalls[d["ID"]] = (st[:5], d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum"),
                       d.get("smsp__inst_executed.sum"))
for (i, k), m in per.items():
    lines.append(f"[{i}] {k}")
    for key in want:
        if key in m:
            lines.append(f"      {key:32s} {m[key]}")
    if i in stalls:
        st, dr, dw, inst = stalls[i]
        lines.append("      stalls per issued instr: " + ", ".join(f"{a}={b:.2f}" for a, b in st))
        lines.append(f"      dram bytes read/write: {dr} / {dw};  warp instructions: {inst}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
