"""Golden parse / solution-file results from the REAL reference (mdroute.bench).

Run in the build container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_formats_golden.py

Writes synthetic Cordeau-layout instance files (generated here, seeded) under
tests/golden/formats/, parses each with the reference's parse_instance (as
every variant the file's type admits, with and without relax_fleet), and
records the resulting instance (dist sha256, labels, scalars, name) plus the
text the reference's write_solution produces for a seeded random solution.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import conftest as rconf  # noqa: E402
from mdroute import bench  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats")


def node_line(rng, fid, windows, combos):
    x, y = rng.uniform(0, 100), rng.uniform(0, 100)
    s, q = rng.choice([0, 5, 10]), rng.randint(1, 30)
    toks = [str(fid), f"{x:.3f}", f"{y:.3f}", str(s), str(q)]
    if combos:
        n = rng.randint(1, 3)
        toks += ["1", str(n)] + [str(2 ** i) for i in range(n)]
    elif windows:  # the window fields follow the (frequency, combo count) pair
        toks += ["1", "0"]
    if windows:
        e = rng.randint(0, 500)
        toks += [str(e), str(e + rng.randint(30, 300))]
    return " ".join(toks)


def make_file(rng, path, ptype, m, n, t, D, Q, windows, combos, shuffle_ids):
    ids = list(range(1, n + 1))
    if shuffle_ids:
        rng.shuffle(ids)
    lines = [f"{ptype} {m} {n} {t}"]
    lines += [f"{D} {Q}" for _ in range(t)]
    lines += [node_line(rng, i, windows, combos) for i in ids]
    for d in range(t):  # depot lines: no demand/service, optional window
        x, y = rng.uniform(0, 100), rng.uniform(0, 100)
        tail = " 0 0 0 0" + (" 0 1000" if windows else "")
        lines.append(f"{n + d + 1} {x:.3f} {y:.3f}{tail}")
    with open(path, "w") as f:
        f.write("\n\n".join(lines[:2]) + "\n" + "\n".join(lines[2:]) + "\n")


def main():
    os.makedirs(HERE, exist_ok=True)
    rng = random.Random(4242)
    files = [
        ("vrp_a.txt", 2, 4, 30, 3, 0, 80, False, True, False),
        ("vrp_b.txt", 2, 0, 25, 2, 200, 60, False, False, True),
        ("tw_a.txt", 6, 3, 24, 2, 0, 100, True, True, True),
        ("tw_b.txt", 6, 2, 18, 3, 900, 0, True, False, False),
    ]
    manifest = {}
    for fname, ptype, m, n, t, D, Q, windows, combos, shuf in files:
        path = os.path.join(HERE, fname)
        make_file(rng, path, ptype, m, n, t, D, Q, windows, combos, shuf)
        variants = ["mdvrptw"] if ptype == 6 else ["mdvrp", "mdovrp"]
        for v in variants:
            for relax in (False, True):
                inst = bench.parse_instance(path, v, relax_fleet=relax)
                sol = rconf.random_solution(random.Random(rng.randrange(1 << 30)), inst)
                out = os.path.join(HERE, f"{fname}.{v}.{int(relax)}.sol")
                bench.write_solution(sol, out, inst)
                back = bench.read_solution(out, inst)
                manifest[f"{fname}|{v}|{int(relax)}"] = dict(
                    dist_sha=hashlib.sha256(np.ascontiguousarray(inst.dist).tobytes()).hexdigest(),
                    labels=list(map(int, inst.labels)), name=inst.name, n_depots=inst.n_depots,
                    fleet=float(inst.fleet_per_depot), capacity=float(inst.capacity),
                    max_duration=float(inst.max_duration),
                    routes=[(r.depart, r.arrive, list(r.customers)) for r in sol.routes],
                    read_back=[(r.depart, r.arrive, list(r.customers)) for r in back.routes],
                    sol_file=os.path.basename(out))
    bad = {
        "empty.txt": "",
        "short_header.txt": "2 4 30\n",
        "bad_header.txt": "2 x 3 1\n0 80\n",
        "too_few_lines.txt": "2 1 3 1\n0 80\n1 1 1 0 1\n",
        "hetero.txt": "2 1 1 2\n0 80\n0 90\n1 1 1 0 1\n2 0 0\n3 5 5\n",
        "no_windows.txt": "6 1 1 1\n0 80\n1 1 1 0 1\n2 0 0\n",
    }
    errors = {}
    for fname, text in bad.items():
        path = os.path.join(HERE, fname)
        with open(path, "w") as f:
            f.write(text)
        v = "mdvrptw" if text.startswith("6") else "mdvrp"
        try:
            bench.parse_instance(path, v)
            errors[fname] = [v, None]
        except bench.ParseError as e:
            errors[fname] = [v, str(e).replace(HERE + "/", "")]
    try:  # wrong problem type for the variant
        bench.parse_instance(os.path.join(HERE, "vrp_a.txt"), "mdvrptw")
    except bench.ParseError as e:
        errors["vrp_a.txt"] = ["mdvrptw", str(e)]
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(dict(cases=manifest, errors=errors), f, indent=0)
    print(len(manifest), "parse cases,", len(errors), "error cases")


if __name__ == "__main__":
    main()
