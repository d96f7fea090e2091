"""Cordeau-format instance files and solution files (mirrors `mdroute.bench`
bench.py:24-156).  Host-side I/O feeding the
device path with real benchmark instances: `parse_instance` builds the same
`Instance` (identical distance matrix, labels, fleet/capacity/duration
relaxations) and `write_solution` / `read_solution` produce and read the same
text.

Layout: a header `type m n t` (vehicles per depot, customers, depots), t lines
`D Q` (0 = unlimited), n customer lines `id x y service demand f a <a combo
fields> [e l]`, then t depot lines in the same layout.
"""
from __future__ import annotations

from pathlib import Path

from .model import INF, Instance, Route, Solution, Variant

EXPECTED_TYPE = {Variant.MDVRP: 2, Variant.MDVRPTW: 6, Variant.MDOVRP: 2}


class ParseError(ValueError):
    pass


def _tokens(path: Path):
    return [(i, ln.split()) for i, ln in enumerate(path.read_text().splitlines(), start=1) if ln.split()]


def _node_fields(lineno, toks, want_windows):
    """(file_id, x, y, service, demand, e, l) of one node line (bench.py:38-56)."""
    try:
        fid = int(float(toks[0]))
        x, y = float(toks[1]), float(toks[2])
        service = float(toks[3]) if len(toks) > 3 else 0.0
        demand = float(toks[4]) if len(toks) > 4 else 0.0
        rest = toks[5:]
        if len(rest) >= 2:
            rest = rest[2 + int(float(rest[1])):]  # skip frequency, combo count and combos
        e = l = None
        if len(rest) >= 2:
            e, l = float(rest[-2]), float(rest[-1])
    except (ValueError, IndexError) as exc:
        raise ParseError(f"line {lineno}: malformed node line: {exc}") from exc
    if want_windows and e is None:
        raise ParseError(f"line {lineno}: time-window fields missing for TW variant")
    return fid, x, y, service, demand, e, l


def parse_instance(path, variant, relax_fleet: bool = False) -> Instance:
    """Parse one instance file and apply the variant's relaxations (bench.py:59-121)."""
    path = Path(path)
    variant = Variant(variant)
    lines = _tokens(path)
    if not lines:
        raise ParseError(f"{path}: empty instance file")
    lineno, head = lines[0]
    if len(head) < 4:
        raise ParseError(f"line {lineno}: header needs 'type m n t'")
    try:
        ptype, m, n, t = (int(float(v)) for v in head[:4])
    except ValueError as exc:
        raise ParseError(f"line {lineno}: bad header: {exc}") from exc
    if ptype != EXPECTED_TYPE[variant]:
        raise ParseError(f"line {lineno}: problem type {ptype} does not match variant {variant.value} "
                         f"(expected {EXPECTED_TYPE[variant]})")
    if len(lines) < 1 + t + n + t:
        raise ParseError(f"{path}: expected {1 + t + n + t} data lines, found {len(lines)}")
    specs = []
    for lineno, toks in lines[1:1 + t]:
        if len(toks) < 2:
            raise ParseError(f"line {lineno}: depot spec needs 'D Q'")
        specs.append((float(toks[0]), float(toks[1])))
    if len({d for d, _ in specs}) > 1 or len({q for _, q in specs}) > 1:
        raise ParseError(f"{path}: heterogeneous depot specs are not supported")
    duration, cap = specs[0]
    capacity = cap if cap > 0 else INF
    max_duration = duration if duration > 0 else INF
    windows = variant is Variant.MDVRPTW
    cust_rows = [_node_fields(ln, tk, windows) for ln, tk in lines[1 + t:1 + t + n]]
    depot_rows = [_node_fields(ln, tk, False) for ln, tk in lines[1 + t + n:1 + t + n + t]]
    fleet = float(m) if m > 0 else INF
    if variant is Variant.MDOVRP:
        fleet, max_duration = INF, INF
    if relax_fleet:
        fleet = INF
    depot_windows = None
    if windows:
        depot_windows = [(r[5] if r[5] is not None else 0.0, r[6] if r[6] is not None else INF)
                         for r in depot_rows]
    customers = [(x, y, q, s, e, l) if windows else (x, y, q, s) for _, x, y, s, q, e, l in cust_rows]
    labels = [r[0] for r in depot_rows] + [r[0] for r in cust_rows]
    return Instance.from_coords(variant, [(r[1], r[2]) for r in depot_rows], customers, fleet_per_depot=fleet,
                                capacity=capacity, max_duration=max_duration, depot_windows=depot_windows,
                                labels=labels, name=path.stem)


def _route_sim(route, inst):
    """(distance, load) of simulate_route (model.py:242-282): sequential sums."""
    seq = route.sequence(inst.open_routes)
    dist = 0.0
    load = 0.0
    for a, b in zip(seq, seq[1:]):
        dist += inst.dist[a, b]
        load += inst.demand[b]
    return float(dist), float(load)


def _route_distance(route, inst):
    seq = route.sequence(inst.open_routes)
    return float(sum(inst.dist[a, b] for a, b in zip(seq, seq[1:])))


def write_solution(sol: Solution, path, inst: Instance) -> None:
    """Total cost, then `depart_label [arrive_label] cost load: c1 c2 ...` per route (bench.py:128-141)."""
    lab = inst.labels
    lines = [f"{sum(_route_distance(r, inst) for r in sol.routes):.2f}"]
    for r in sol.routes:
        dist, load = _route_sim(r, inst)
        custs = " ".join(str(lab[c]) for c in r.customers)
        if inst.open_routes:
            lines.append(f"{lab[r.depart]} {dist:.2f} {load:g}: {custs}")
        else:
            lines.append(f"{lab[r.depart]} {lab[r.arrive]} {dist:.2f} {load:g}: {custs}")
    Path(path).write_text("\n".join(lines) + "\n")


def read_solution(path, inst: Instance) -> Solution:
    """Inverse of write_solution (bench.py:144-156)."""
    label_to_id = {lab: i for i, lab in enumerate(inst.labels)}
    lines = [ln for ln in Path(path).read_text().splitlines() if ln.strip()]
    sol = Solution()
    for ln in lines[1:]:
        head, _, tail = ln.partition(":")
        toks = head.split()
        custs = [label_to_id[int(v)] for v in tail.split()]
        depart = label_to_id[int(toks[0])]
        arrive = depart if inst.open_routes else label_to_id[int(toks[1])]
        sol.routes.append(Route(depart, arrive, custs))
    return sol
