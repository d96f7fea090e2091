"""Problem data model mirrored from the reference (`mdroute.model`).

Only what the local-search path consumes is kept: `Instance` arrays and flags
(model.py:39-154), `Route` (model.py:157-177) and `Solution` (model.py:180-202).
Every entry point of this package is duck-typed on these attribute names, so
the reference package's own `Instance` / `Solution` objects can be passed in
unchanged (drop-in use).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import Optional

import numpy as np

INF = math.inf


class Variant(str, Enum):
    """model.py:19-22"""

    MDVRP = "mdvrp"
    MDVRPTW = "mdvrptw"
    MDOVRP = "mdovrp"


@dataclass(frozen=True)
class Node:
    id: int
    kind: str
    x: float
    y: float
    demand: float = 0.0
    service: float = 0.0
    tw_early: float = 0.0
    tw_late: float = INF


class Instance:
    """Immutable problem data; depots are node ids 0..n_depots-1 (model.py:39-108)."""

    def __init__(self, variant, nodes, n_depots, dist, time=None, fleet_per_depot=INF,
                 capacity=INF, max_duration=INF, labels=None, name=""):
        self.variant = Variant(variant)
        self.nodes = nodes
        self.n_depots = int(n_depots)
        self.n_customers = len(nodes) - self.n_depots
        if self.n_depots < 1 or self.n_customers < 1:
            raise ValueError("instance needs at least one depot and one customer")
        self.dist = np.ascontiguousarray(dist, dtype=np.float64)
        self.time = self.dist if time is None else np.ascontiguousarray(time, dtype=np.float64)
        n = len(nodes)
        for m, what in ((self.dist, "distance"), (self.time, "time")):
            if m.shape != (n, n):
                raise ValueError(f"{what} matrix shape {m.shape} does not match node count")
            if np.abs(np.diag(m)).max() > 1e-12 or not np.allclose(m, m.T, atol=1e-9):
                raise ValueError(f"{what} matrix must be symmetric with zero diagonal")
        self.fleet_per_depot = fleet_per_depot
        self.capacity = capacity
        self.max_duration = max_duration
        self.open_routes = self.variant is Variant.MDOVRP
        self.labels = labels if labels is not None else list(range(n))
        self.name = name
        self.demand = np.array([nd.demand for nd in nodes], dtype=np.float64)
        self.service = np.array([nd.service for nd in nodes], dtype=np.float64)
        self.tw_early = np.array([nd.tw_early for nd in nodes], dtype=np.float64)
        self.tw_late = np.array([nd.tw_late for nd in nodes], dtype=np.float64)
        self.xy = np.array([[nd.x, nd.y] for nd in nodes], dtype=np.float64)
        for nd in nodes:
            if nd.demand < 0:
                raise ValueError(f"node {nd.id}: negative demand")
            if nd.tw_early > nd.tw_late:
                raise ValueError(f"node {nd.id}: empty time window")
        for d in range(self.n_depots):
            if nodes[d].demand != 0 or nodes[d].service != 0:
                raise ValueError(f"depot {d}: demand and service must be zero")

    @property
    def n_nodes(self) -> int:
        return len(self.nodes)

    @property
    def has_windows(self) -> bool:
        return self.variant is Variant.MDVRPTW

    def depots(self) -> range:
        return range(self.n_depots)

    def customers(self) -> range:
        return range(self.n_depots, self.n_nodes)

    def is_depot(self, node: int) -> bool:
        return 0 <= node < self.n_depots

    @staticmethod
    def from_coords(variant, depot_xy, customers, fleet_per_depot=INF, capacity=INF,
                    max_duration=INF, depot_windows=None, labels=None, name="") -> "Instance":
        """Euclidean instance; travel time = distance (model.py:110-154).

        Customer tuples are (x, y, demand[, service[, e, l]]).
        """
        nodes: list[Node] = []
        for d, (x, y) in enumerate(depot_xy):
            e, l = (0.0, INF) if depot_windows is None else depot_windows[d]
            nodes.append(Node(d, "depot", float(x), float(y), 0.0, 0.0, e, l))
        base = len(depot_xy)
        for i, c in enumerate(customers):
            s = c[3] if len(c) > 3 else 0.0
            e, l = (c[4], c[5]) if len(c) > 5 else (0.0, INF)
            nodes.append(Node(base + i, "customer", float(c[0]), float(c[1]), float(c[2]),
                              float(s), float(e), float(l)))
        xy = np.array([[nd.x, nd.y] for nd in nodes])
        dx = xy[:, 0][:, None] - xy[:, 0][None, :]
        dy = xy[:, 1][:, None] - xy[:, 1][None, :]
        # (dx*dx + dy*dy): the same rounding as a length-2 numpy pairwise sum
        dist = np.sqrt(dx * dx + dy * dy)
        np.fill_diagonal(dist, 0.0)
        return Instance(Variant(variant), nodes, len(depot_xy), dist,
                        fleet_per_depot=fleet_per_depot, capacity=capacity,
                        max_duration=max_duration, labels=labels, name=name)


class Route:
    """Depot endpoints plus an ordered customer list (model.py:157-177)."""

    __slots__ = ("depart", "arrive", "customers", "attr")

    def __init__(self, depart: int, arrive: int, customers: Optional[list] = None, attr=None):
        self.depart = depart
        self.arrive = arrive
        self.customers = customers if customers is not None else []
        self.attr = attr

    def sequence(self, open_routes: bool) -> list:
        if open_routes:
            return [self.depart] + self.customers
        return [self.depart] + self.customers + [self.arrive]

    def clone(self) -> "Route":
        return Route(self.depart, self.arrive, list(self.customers), self.attr)

    def __repr__(self) -> str:
        return f"Route({self.depart}->{self.arrive}, {self.customers})"


class Solution:
    """Ordered route list; route order is part of the tie-break key (model.py:180-202)."""

    __slots__ = ("routes", "meta")

    def __init__(self, routes=None, meta=None):
        self.routes = routes if routes is not None else []
        self.meta = meta if meta is not None else {}

    def clone(self) -> "Solution":
        return Solution([r.clone() for r in self.routes], dict(self.meta))

    def customer_list(self) -> list:
        out: list = []
        for r in self.routes:
            out.extend(r.customers)
        return out

    def drop_empty_routes(self) -> None:
        self.routes = [r for r in self.routes if r.customers]

    def __repr__(self) -> str:
        return f"Solution({len(self.routes)} routes)"


def route_edges(route, open_routes: bool) -> set:
    """Undirected arcs of a route, the return arc omitted when open (model.py:217-220)."""
    seq = route.sequence(open_routes)
    return {(a, b) if a <= b else (b, a) for a, b in zip(seq, seq[1:])}


def solution_edges(sol, open_routes: bool) -> set:
    out: set = set()
    for r in sol.routes:
        if r.customers:
            out |= route_edges(r, open_routes)
    return out


def route_distance(route, inst) -> float:
    seq = route.sequence(inst.open_routes)
    d = inst.dist
    return float(sum(d[a, b] for a, b in zip(seq, seq[1:])))


def flatten(sol):
    """Solution -> (off[m+1], cust, depart[m], arrive[m]) int32 arrays."""
    routes = sol.routes
    m = len(routes)
    off = np.zeros(m + 1, dtype=np.int32)
    if m:
        np.cumsum([len(r.customers) for r in routes], out=off[1:])
    cust = np.fromiter((c for r in routes for c in r.customers), dtype=np.int32, count=int(off[-1]))
    dep = np.array([r.depart for r in routes], dtype=np.int32)
    arr = np.array([r.arrive for r in routes], dtype=np.int32)
    return off, cust, dep, arr


def unflatten(off, cust, dep, arr, route_cls=Route):
    return [route_cls(int(dep[r]), int(arr[r]), [int(c) for c in cust[off[r]:off[r + 1]]])
            for r in range(len(dep))]
