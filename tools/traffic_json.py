"""profiles/r1_traffic.json from a full-set capture of one evaluation phase's launches (per-kernel DRAM bytes)."""
import collections, csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
units = rows[1]
k = collections.defaultdict(lambda: {"launches": 0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0})
for r in rows[2:]:
    name = r[ik].split("(")[0].replace("void ", "").replace("mdr::", "")
    k[name]["launches"] += 1
    k[name]["dram_read_bytes"] += float(r[ir].replace(",", "")) * unit.get(units[ir], 1)
    k[name]["dram_write_bytes"] += float(r[iw].replace(",", "")) * unit.get(units[iw], 1)
n = sum(v["launches"] for v in k.values())
tot = sum(v["dram_read_bytes"] + v["dram_write_bytes"] for v in k.values())
json.dump({"source": sys.argv[3] if len(sys.argv) > 3 else rep, "launches_captured": n, "kernels": k,
           "evaluation_phase_dram_bytes_per_round": tot / 2}, open(out, "w"), indent=1)
print(n, tot / 2)
