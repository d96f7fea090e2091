"""Cordeau benchmark files: instance parsing and solution files (SURVEY.md
sec. 8(f) row 4; drop-in for `mdroute.bench.parse_instance`, `write_solution`
and `read_solution`, bench.py:24-156).

The instance reader walks the non-blank lines with a cursor through three
sections -- header `type m n t`, t depot specs `D Q`, n customer records and
t depot records (`id x y service demand [f a combos...] [e l]`) -- and hands
the coordinates to `Instance.from_coords`, so the distance matrix, labels and
relaxations (fleet 0 = unlimited, MDOVRP without fleet and duration limits,
`relax_fleet`) equal the reference's, and so do the error messages.  A
solution file's per-route distance and load come from the device route
simulation (mdr_route_sim, the same sequential sums as simulate_route).
"""
from __future__ import annotations

from pathlib import Path

from .model import INF, Instance, Route, Solution, Variant

EXPECTED_TYPE = {Variant.MDVRP: 2, Variant.MDVRPTW: 6, Variant.MDOVRP: 2}


class ParseError(ValueError):
    pass


class _Lines:
    """Non-blank lines of a file as (line number, tokens), consumed in order."""

    def __init__(self, path: Path):
        self.rows = [(no, ln.split()) for no, ln in enumerate(path.read_text().splitlines(), 1) if ln.strip()]
        self.at = 0

    def take(self, k: int):
        out = self.rows[self.at:self.at + k]
        self.at += k
        return out


class _Record:
    """One node line: file id, coordinates, service, demand and the optional window."""

    __slots__ = ("fid", "x", "y", "service", "demand", "window")

    def __init__(self, lineno: int, toks, need_window: bool):
        try:
            self.fid = int(float(toks[0]))
            self.x, self.y = float(toks[1]), float(toks[2])
            self.service = float(toks[3]) if len(toks) > 3 else 0.0
            self.demand = float(toks[4]) if len(toks) > 4 else 0.0
            tail = toks[5:]
            if len(tail) >= 2:  # visit frequency, combination count, the combinations
                tail = tail[2 + int(float(tail[1])):]
            self.window = (float(tail[-2]), float(tail[-1])) if len(tail) >= 2 else None
        except (ValueError, IndexError) as exc:
            raise ParseError(f"line {lineno}: malformed node line: {exc}") from exc
        if need_window and self.window is None:
            raise ParseError(f"line {lineno}: time-window fields missing for TW variant")


def parse_instance(path, variant, relax_fleet: bool = False) -> Instance:
    """Read a Cordeau instance file for `variant` (bench.py:59-121)."""
    path, variant = Path(path), Variant(variant)
    src = _Lines(path)
    if not src.rows:
        raise ParseError(f"{path}: empty instance file")
    (hline, head), = src.take(1)
    if len(head) < 4:
        raise ParseError(f"line {hline}: header needs 'type m n t'")
    try:
        ptype, vehicles, n_cust, n_dep = (int(float(v)) for v in head[:4])
    except ValueError as exc:
        raise ParseError(f"line {hline}: bad header: {exc}") from exc
    want = EXPECTED_TYPE[variant]
    if ptype != want:
        raise ParseError(f"line {hline}: problem type {ptype} does not match variant {variant.value} "
                         f"(expected {want})")
    need = 1 + 2 * n_dep + n_cust
    if len(src.rows) < need:
        raise ParseError(f"{path}: expected {need} data lines, found {len(src.rows)}")

    specs = set()
    for lineno, toks in src.take(n_dep):
        if len(toks) < 2:
            raise ParseError(f"line {lineno}: depot spec needs 'D Q'")
        specs.add((float(toks[0]), float(toks[1])))
    durations, capacities = {d for d, _ in specs}, {q for _, q in specs}
    if len(durations) > 1 or len(capacities) > 1:
        raise ParseError(f"{path}: heterogeneous depot specs are not supported")
    duration, = durations
    cap, = capacities

    tw = variant is Variant.MDVRPTW
    cust = [_Record(no, tk, tw) for no, tk in src.take(n_cust)]
    deps = [_Record(no, tk, False) for no, tk in src.take(n_dep)]

    limits = dict(fleet_per_depot=float(vehicles) if vehicles > 0 else INF,
                  capacity=cap if cap > 0 else INF,
                  max_duration=duration if duration > 0 else INF)
    if variant is Variant.MDOVRP:
        limits.update(fleet_per_depot=INF, max_duration=INF)
    if relax_fleet:
        limits["fleet_per_depot"] = INF
    if tw:
        customers = [(c.x, c.y, c.demand, c.service, *c.window) for c in cust]
        windows = [d.window if d.window is not None else (0.0, INF) for d in deps]
    else:
        customers = [(c.x, c.y, c.demand, c.service) for c in cust]
        windows = None
    return Instance.from_coords(variant, [(d.x, d.y) for d in deps], customers, depot_windows=windows,
                                labels=[r.fid for r in deps + cust], name=path.stem, **limits)


def write_solution(sol: Solution, path, inst: Instance, device: int = 0) -> None:
    """Total cost, then `depart_label [arrive_label] cost load: c1 c2 ...` per route
    (bench.py:128-141); distances and loads from the device route simulation."""
    from .feasibility import _simulate
    sims = _simulate(sol.routes, inst, False, device)
    lab = inst.labels
    total = 0
    for row in sims:
        total += float(row[0])
    out = [f"{total:.2f}"]
    for r, row in zip(sol.routes, sims):
        ends = f"{lab[r.depart]}" if inst.open_routes else f"{lab[r.depart]} {lab[r.arrive]}"
        out.append(f"{ends} {float(row[0]):.2f} {float(row[1]):g}: " + " ".join(str(lab[c]) for c in r.customers))
    Path(path).write_text("\n".join(out) + "\n")


def read_solution(path, inst: Instance) -> Solution:
    """Routes of a solution file, labels mapped back to node ids (bench.py:144-156)."""
    node_of = {lab: i for i, lab in enumerate(inst.labels)}
    sol = Solution()
    body = [ln for ln in Path(path).read_text().splitlines() if ln.strip()][1:]
    for ln in body:
        ends, _, members = ln.partition(":")
        ids = ends.split()
        dep = node_of[int(ids[0])]
        arr = dep if inst.open_routes else node_of[int(ids[1])]
        sol.routes.append(Route(dep, arr, [node_of[int(v)] for v in members.split()]))
    return sol
