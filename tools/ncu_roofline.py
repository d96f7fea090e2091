"""Binding-roof summary of a config's dominant evaluator from an ncu --set full capture.

    python tools/ncu_roofline.py CONFIG REPORT.ncu-rep [KERNEL_REGEX [LABEL]]
        -> merges profiles/ncu_roofline.json[CONFIG][LABEL] (LABEL default "relocate")

For every captured launch of the kernel (default: the relocate staged
evaluator, k_eval_c<*, 0, *, *>) it reads the utilisation of each SM-side roof
ncu reports -- instruction issue, the FP64 pipe, L1/TEX, L2 (lts), DRAM -- and
names the highest one the binding roof.  bench.py quotes the entry of its
config in roofline{bound, achieved, peak, frac, traffic}.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name in the json, ncu metric, scale to a 0..1 fraction)
ROOFS = [
    ("issue", "sm__inst_issued.avg.pct_of_peak_sustained_active", 0.01),
    ("fp64_pipe", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.01),
    ("l1tex", "l1tex__throughput.avg.pct_of_peak_sustained_active", 0.01),
    ("l2", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 0.01),
    ("dram", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0.01),
]
EXTRA = {
    "duration_ns": "gpu__time_duration.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issued_per_scheduler_cycle": "smsp__issue_active.avg.per_cycle_active",
    "warp_inst": "smsp__inst_executed.sum",
    "fp64_pipe_elapsed_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "lts_sectors": "lts__t_sectors.sum",
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "ns": 1.0, "usecond": 1e3,
         "us": 1e3, "msecond": 1e6, "ms": 1e6}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    cfg, rep = sys.argv[1], sys.argv[2]
    kre = re.compile(sys.argv[3] if len(sys.argv) > 3 else r"k_eval_c<[^,]+, 0, \d+, \d+(, \d+)?>")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    kcol = col.get("Kernel Name")
    launches = []
    for r in rows[2:]:  # row 1: units
        if len(r) != len(hdr) or not kre.search(r[kcol]):
            continue
        m = {}
        for name, met, sc in ROOFS:
            v = num(r[col[met]]) if met in col else None
            m[name] = None if v is None else v * sc
        for name, met in EXTRA.items():
            v = num(r[col[met]]) if met in col else None
            m[name] = None if v is None else v * SCALE.get(units[col[met]], 1.0)
        m["kernel"] = r[kcol]
        launches.append(m)
    if not launches:
        sys.exit(f"no launch of {kre.pattern} in {rep}")
    n = len(launches)
    avg = {k: (sum(x[k] for x in launches if x[k] is not None) / max(1, sum(1 for x in launches if x[k] is not None))
               if any(x[k] is not None for x in launches) else None)
           for k in launches[0] if k != "kernel"}
    roofs = {k: avg[k] for k, _, _ in ROOFS if avg.get(k) is not None}
    binding = max(roofs, key=roofs.get)
    traffic = None
    if avg.get("dram_read") is not None and avg.get("dram_write") is not None:
        traffic = avg["dram_read"] + avg["dram_write"]
    entry = {"kernel": launches[0]["kernel"], "launches_averaged": n, "binding": binding,
             "achieved": roofs[binding], "peak": 1.0, "unit": "fraction of the ncu peak of that unit",
             "frac": roofs[binding], "roofs": roofs, "dram_bytes_per_launch": traffic,
             "metrics": {k: v for k, v in avg.items() if k not in roofs},
             "source": os.path.relpath(rep, ROOT)}
    path = os.environ.get("NCU_ROOFLINE_OUT") or os.path.join(ROOT, "profiles", "ncu_roofline.json")
    allj = json.load(open(path)) if os.path.exists(path) else {}
    label = sys.argv[4] if len(sys.argv) > 4 else "relocate"
    if not isinstance(allj.get(cfg), dict) or "binding" in allj.get(cfg, {}):
        allj[cfg] = {}
    allj[cfg][label] = entry
    json.dump(allj, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
