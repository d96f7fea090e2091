"""Scalar restatement of the reference's population management -- TEST
INFRASTRUCTURE ONLY (the checker of csrc/mdr_population.cu; never on the
product path).

Follows population.py:19-34 (solution_distance, population_distance),
51-67 (biased_fitness) and 94-116 (distance matrix, survivor_selection) of
/root/reference/pkg/src/mdroute, on edge sets given as sorted key arrays.
Pinned to the reference by tests/golden/population.json
(tests/golden/make_population_golden.py).
"""
from __future__ import annotations


def edge_distance(a, b) -> float:
    """population.py:19-24 on key arrays (intersection by a two-pointer merge)."""
    if len(a) == 0 and len(b) == 0:
        return 0.0
    i = j = inter = 0
    while i < len(a) and j < len(b):
        if a[i] == b[j]:
            inter += 1
            i += 1
            j += 1
        elif a[i] < b[j]:
            i += 1
        else:
            j += 1
    return 100.0 * (1.0 - inter / max(len(a), len(b)))


def distance_rows(edges):
    n = len(edges)
    rows = [[0.0] * n for _ in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            rows[i][j] = rows[j][i] = edge_distance(edges[i], edges[j])
    return rows


def nearest_mean(i, rows, alive):
    """population.py:27-34: mean of the 5 smallest distances to the other members."""
    ds = sorted(rows[i][j] for j in alive if j != i)[:5]
    return sum(ds) / len(ds) if ds else 0.0


def removal_order(edges, costs, births, mu, xi):
    """Indices removed by survivor_selection (population.py:103-116), in order."""
    rows = distance_rows(edges)
    alive = list(range(len(edges)))
    out = []
    while len(alive) > mu:
        n = len(alive)
        div = {i: nearest_mean(i, rows, alive) for i in alive}
        by_f = sorted(alive, key=lambda i: (costs[i], births[i]))
        by_d = sorted(alive, key=lambda i: (-div[i], births[i]))
        rf = {i: r for r, i in enumerate(by_f)}
        rd = {i: r for r, i in enumerate(by_d)}
        chi = {i: (n - rf[i]) / n + xi * (n - rd[i]) / n for i in alive}
        worst = min(alive, key=lambda i: (chi[i], births[i]))
        out.append(worst)
        alive.remove(worst)
    return out
