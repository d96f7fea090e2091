import csv, io, subprocess, sys
rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h = raw[0]
for row in raw[2:]:
    d = dict(zip(h, row))
    st = sorted([(k, float(d[k])) for k in h if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")], key=lambda x: -x[1])
    print(d["Kernel Name"][:22], "inst=%.3g" % float(d["smsp__inst_executed.sum"]), " ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in st[:6]))
