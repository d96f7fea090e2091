"""Summarise an ncu report: SOL, occupancy, stalls, instruction mix, hot source lines."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]


def q(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(q("--page", "details", "--csv"))))
h = det[0]
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Section Name") in ("GPU Speed Of Light Throughput", "Occupancy", "Scheduler Statistics",
                                 "Warp State Statistics", "Launch Statistics") and d.get("Metric Name") in (
            "Duration", "Compute (SM) Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
            "L2 Cache Throughput", "DRAM Throughput", "Achieved Occupancy", "Registers Per Thread",
            "Issued Warp Per Scheduler", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
            "Theoretical Occupancy"):
        print(f"{d['Metric Name']:36s} {d['Metric Value']} {d.get('Metric Unit', '')}")
raw = list(csv.reader(io.StringIO(q("--page", "raw", "--csv"))))
h, u, r = raw[0], raw[1], raw[2]
d = dict(zip(h, r))
st = sorted([(k, float(d[k])) for k in h if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")],
            key=lambda x: -x[1])
print("stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in st[:7]))
print("inst executed (warp):", d.get("smsp__inst_executed.sum"))
sass = list(csv.reader(io.StringIO(q("--page", "source", "--csv", "--print-source=sass"))))
hh = sass[1]
ix, ie = hh.index("Source"), hh.index("Instructions Executed")
cnt = collections.Counter()
tot = 0
for row in sass[2:]:
    try:
        n = float(row[ie] or 0)
    except (ValueError, IndexError):
        continue
    t = row[ix].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    cnt[op] += n
    tot += n
print("mix:", ", ".join(f"{k}={v / tot * 100:.1f}%" for k, v in cnt.most_common(12)))
src = list(csv.reader(io.StringIO(q("--page", "source", "--csv", "--print-source=cuda"))))
# cuda view: find header with 'Instructions Executed'
lines = []
hdr = None
fname = None
for row in src:
    if row and row[0] == "File Name":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if hdr and len(row) == len(hdr) and "Instructions Executed" in hdr:
        try:
            n = float(row[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        if n > 0:
            lines.append((n, fname, row[0], row[1].strip()[:90]))
lines.sort(reverse=True)
print("hot lines (warp inst executed):")
for n, f, ln, s in lines[:25]:
    print(f"  {n / tot * 100:5.1f}%  {f}:{ln}  {s}")
