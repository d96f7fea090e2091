"""Population sharding across GPUs and the periodic elite exchange.

Individuals are independent, so the population is split into
contiguous shards, one per rank, with the instance replicated; the local
search itself has no data-path collective.  The only collective is the
periodic exchange of elite solutions: every rank encodes its best solution as
a fixed-size int32 vector and `all_gather`s it (NCCL over NVLink on the GPU
path, gloo in the CPU tests).

Encoding (length n_customers + 3*J + 2):
    [n_routes, D_bits_hi, (depart, arrive, k, customers...) per route, -1 padding]
where D is the solution's distance stored as the two 32-bit halves of its IEEE
bits (so the elite's cost travels exactly).
"""
from __future__ import annotations

import struct

import numpy as np


def shard_range(n_total: int, world: int, rank: int) -> range:
    """Contiguous shard of individual ids for `rank` (remainder spread over the first ranks)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def encode_len(n_customers: int, J: int) -> int:
    return n_customers + 3 * J + 3


def encode_elite(routes, D: float, n_customers: int, J: int) -> np.ndarray:
    """routes: [(depart, arrive, customers)]."""
    out = np.full(encode_len(n_customers, J), -1, dtype=np.int32)
    if len(routes) > J:
        raise ValueError("more routes than the encoding capacity J")
    bits = struct.unpack("<II", struct.pack("<d", float(D)))
    out[0] = len(routes)
    out[1] = np.int32(np.uint32(bits[0]).view(np.int32))
    out[2] = np.int32(np.uint32(bits[1]).view(np.int32))
    at = 3
    for dep, arr, cust in routes:
        out[at:at + 3] = (dep, arr, len(cust))
        at += 3
        out[at:at + len(cust)] = cust
        at += len(cust)
    return out


def decode_elite(vec):
    v = np.asarray(vec, dtype=np.int32)
    m = int(v[0])
    bits = (int(np.int32(v[1]).view(np.uint32)), int(np.int32(v[2]).view(np.uint32)))
    D = struct.unpack("<d", struct.pack("<II", *bits))[0]
    routes = []
    at = 3
    for _ in range(m):
        dep, arr, k = (int(x) for x in v[at:at + 3])
        at += 3
        routes.append((dep, arr, [int(x) for x in v[at:at + k]]))
        at += k
    return routes, D


def exchange_elites(local_vec, group=None, device=None):
    """all_gather of every rank's encoded elite; returns a list of numpy vectors (rank order)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.asarray(local_vec, dtype=np.int32))
    if device is not None:
        t = t.to(device)
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    return [b.cpu().numpy() for b in bufs]


def best_of(elites):
    """Index and decoded routes of the lowest-D elite (ties: lowest rank)."""
    best = None
    for i, e in enumerate(elites):
        routes, D = decode_elite(e)
        if best is None or D < best[2]:
            best = (i, routes, D)
    return best
