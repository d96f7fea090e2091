"""Hot source lines of one kernel in an ncu report: python tools/ncu_lines.py REP SKIP [N]"""
import csv, io, subprocess, sys, collections
rep, skip = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
fpath = None
cur = None
hdr = None
agg = collections.Counter()
stall = collections.Counter()
src = {}
tot = 0
stot = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fpath = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr):
        continue
    try:
        ie = hdr.index("Instructions Executed")
        n = float(row[ie] or 0)
        s = float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    if not row[0].strip():
        continue
    key = (fpath, int(row[0]))
    src[key] = row[1].strip()[:80]
    agg[key] += n
    stall[key] += s
    tot += n
    stot += s
print("total warp inst %.3g" % tot)
order = sys.argv[4] if len(sys.argv) > 4 else "stall"
for key, n in sorted(agg.items(), key=lambda kv: -(stall[kv[0]] if order == "stall" else kv[1]))[:top]:
    print(f"{n / tot * 100:5.1f}% inst {stall[key] / stot * 100:5.1f}% stall  {key[0]}:{key[1]:<4d} {src[key]}")
