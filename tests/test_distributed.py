"""Multi-process (gloo, world_size 2, CPU) tests of the sharding and elite-exchange host logic."""
import os
import random
import socket

import torch.multiprocessing as mp

from paper_2605_05208_b200 import distributed as D
from paper_2605_05208_b200 import workload as W


def test_shard_range_partitions_population():
    for n in (1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            ids = [i for r in range(world) for i in D.shard_range(n, world, r)]
            assert ids == list(range(n))


def test_encode_decode_round_trip_exact():
    inst = W.make_instance(random.Random(3), "mdvrp", n_customers=30, n_depots=3)
    sol = W.random_solution(random.Random(4), inst)
    routes = [(r.depart, r.arrive, list(r.customers)) for r in sol.routes]
    v = D.encode_elite(routes, 1234.5678901234567, inst.n_customers, len(routes) + 5)
    got, d = D.decode_elite(v)
    assert got == routes and d == 1234.5678901234567


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = W.make_instance(random.Random(5), "mdvrptw", n_customers=25, n_depots=2)
    ids = list(D.shard_range(6, world, rank))
    sols = [W.random_solution(random.Random(100 + i), inst) for i in ids]
    # each rank's elite: its first individual, with a rank-dependent cost
    routes = [(r.depart, r.arrive, list(r.customers)) for r in sols[0].routes]
    v = D.encode_elite(routes, 100.0 - rank, inst.n_customers, 32)
    elites = D.exchange_elites(v)
    best = D.best_of(elites)
    q.put((rank, ids, [D.decode_elite(e)[1] for e in elites], best[0], best[1]))
    dist.destroy_process_group()


def test_gloo_world2_elite_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ids0, costs0, b0, routes0), (r1, ids1, costs1, b1, routes1) = res
    assert ids0 == [0, 1, 2] and ids1 == [3, 4, 5]
    assert costs0 == costs1 == [100.0, 99.0]
    assert b0 == b1 == 1 and routes0 == routes1
    inst = W.make_instance(random.Random(5), "mdvrptw", n_customers=25, n_depots=2)
    want = W.random_solution(random.Random(103), inst)
    assert routes1 == [(r.depart, r.arrive, list(r.customers)) for r in want.routes]
