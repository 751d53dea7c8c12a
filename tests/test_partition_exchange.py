"""The multi-GPU exchange protocol executed across processes (
partition.hpp): 2- and 3-rank gloo groups on CPU, each rank computing the
ADMM phases with the C restatement of the reference (oracle/) on its own copy
of the state, exchanging ONLY the rows of the library's exchange plan
(gridadmm_network_exchange_rows):

  after the branch phase   x of the to-side rows of cut branches  -> to-bus part
  after the bus/z/y phases xbar, z, y of those rows               -> branch part
  every iteration          max-all-reduce of the residual norms.

Every row, branch and bus a rank does not own (and does not mirror through
the plan) is overwritten with NaN before every iteration, so any missing
exchange would poison an owned value.  The owned values and the norm series
must equal a single-process run bit for bit: the plan is sufficient, the
partition cannot change a bit, which is what the NCCL engine (dist.cpp) relies
on.  The GPU side of the same claim is tests/test_partition.py."""
import os
import socket

import numpy as np
import pytest

from conftest import REPO, case_path

CFG = dict(rho_pq=100.0, rho_va=1e4, eps=1e-5, max_inner=1000)
ITERS = 12
ROWF = ("x", "xbar", "z", "y", "lambda")


def ownership(ex, part):
    ng, nb = len(ex["gen"]), len(ex["bus"])
    nl = len(ex["ends"])
    row_owner = np.zeros(2 * ng + 8 * nl, dtype=np.int64)
    for g, row in enumerate(ex["gen"]):
        row_owner[2 * g] = row_owner[2 * g + 1] = part[int(row[0])]
    br_owner = np.zeros(nl, dtype=np.int64)
    for b, (f, t) in enumerate(ex["ends"]):
        base = 2 * ng + 8 * b
        row_owner[[base + 0, base + 1, base + 4, base + 5]] = part[f]
        row_owner[[base + 2, base + 3, base + 6, base + 7]] = part[t]
        br_owner[b] = part[f]
    return row_owner, br_owner, np.asarray(part[:nb])


def norms(s, xbar_prev, z_prev, rows):
    r = s["x"][rows] - s["xbar"][rows] + s["z"][rows]
    return np.array([np.max(np.abs(r), initial=0.0),
                     np.max(np.abs(s["xbar"][rows] - xbar_prev[rows]), initial=0.0),
                     np.max(np.abs(s["z"][rows]), initial=0.0),
                     np.max(np.abs(s["z"][rows] - z_prev[rows]), initial=0.0)])


def heavy_tailed_weights(nl, seed=7):
    """Per-branch weights shaped like measured TRON step counts (a few very
    long chains), for the weighted partition."""
    rng = np.random.default_rng(seed)
    return (rng.pareto(1.2, nl) * 8).astype(np.int32)


def _rank_main(rank, world, path, port, out, weights=None):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, REPO)
    import oracle
    import paper_2110_06879_b200 as ga
    net = ga.Network(path)
    if weights is not None:
        net.set_branch_weights(weights)
    ex = net.export()
    part = net.partition(world)
    row_owner, br_owner, bus_owner = ownership(ex, part)
    plan = {q: net.exchange_rows(world, rank, q) for q in range(world) if q != rank}
    mirror = np.concatenate([plan[q][0] for q in plan]) if plan else np.zeros(0, np.int64)
    own_rows = np.nonzero(row_owner == rank)[0]
    keep_rows = np.zeros(len(row_owner), bool)
    keep_rows[own_rows] = True
    keep_rows[mirror] = True
    port_net = oracle.PortNet(path)
    s = port_net.cold_start(**CFG)  # every rank starts from the full cold start (as Session does)

    def poison():
        for f in ROWF:
            s[f][~keep_rows] = np.nan
        s["x"][~(row_owner == rank)] = np.nan  # x of a mirrored row is recomputed by its branch
        nb = len(bus_owner)
        s["bus_w"][bus_owner != rank] = np.nan
        s["bus_theta"][bus_owner != rank] = np.nan
        nl = len(br_owner)
        bp = s["branch_point"].reshape(nl, 6)
        bp[br_owner != rank] = np.nan
        for f in ("lt_ij", "lt_ji", "rho_tilde"):
            s[f][br_owner != rank] = np.nan
        assert nb > 0

    def exchange(fields, rows_out_idx, rows_in_idx):
        # rows_out_idx(q) -> rows this rank sends to q; rows_in_idx(q) -> rows it receives
        payload = {q: {f: s[f][rows_out_idx(q)].copy() for f in fields} for q in plan}
        box = [None] * world
        dist.all_gather_object(box, payload)
        for q in plan:
            got = box[q][rank]
            for f in fields:
                s[f][rows_in_idx(q)] = got[f]

    series = []
    for _ in range(ITERS):
        poison()
        xbar_prev, z_prev = s["xbar"].copy(), s["z"].copy()
        port_net.phase(0, s, **CFG)
        port_net.phase(1, s, **CFG)
        exchange(("x",), lambda q: plan[q][0], lambda q: plan[q][1])
        for p in (2, 3, 4):
            port_net.phase(p, s, **CFG)
        exchange(("xbar", "z", "y"), lambda q: plan[q][1], lambda q: plan[q][0])
        t = torch.from_numpy(norms(s, xbar_prev, z_prev, own_rows))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        series.append(t.numpy().copy())
    mine = {f: s[f][own_rows].copy() for f in ("x", "xbar", "z", "y")}
    mine["bus_w"] = s["bus_w"][bus_owner == rank].copy()
    mine["branch_point"] = s["branch_point"].reshape(-1, 6)[br_owner == rank].copy()
    out[rank] = {"series": np.array(series), "state": mine, "own_rows": own_rows,
                 "n_mirror": int(len(mirror))}
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,weighted", [("case118", 2, False), ("case118", 3, False),
                                                 ("case30", 2, False), ("case118", 3, True)])
def test_exchange_protocol_bit_identical(gridadmm, oracle_mod, name, world, weighted):
    import torch.multiprocessing as mp
    path = case_path(name)
    net = gridadmm.Network(path)
    weights = None
    if weighted:  # measured-cost partition (gridadmm_network_set_branch_weights)
        unweighted = net.partition(world)
        weights = heavy_tailed_weights(net.num_branches)
        net.set_branch_weights(weights)
        assert not np.array_equal(net.partition(world), unweighted)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    out = mp.Manager().dict()
    mp.spawn(_rank_main, args=(world, path, port, out, weights), nprocs=world, join=True)

    # single process, same phases
    ex = net.export()
    part = net.partition(world)
    row_owner, br_owner, bus_owner = ownership(ex, part)
    port_net = oracle_mod.PortNet(path)
    s = port_net.cold_start(**CFG)
    series = []
    all_rows = np.arange(len(row_owner))
    for _ in range(ITERS):
        xbar_prev, z_prev = s["xbar"].copy(), s["z"].copy()
        for p in range(5):
            port_net.phase(p, s, **CFG)
        series.append(norms(s, xbar_prev, z_prev, all_rows))
    series = np.array(series)
    assert sum(out[r]["n_mirror"] for r in range(world)) > 0  # the partition cuts branches
    for r in range(world):
        got = out[r]
        assert np.array_equal(got["series"].view(np.uint64), series.view(np.uint64)), r
        rows = got["own_rows"]
        for f in ("x", "xbar", "z", "y"):
            assert np.array_equal(got["state"][f].view(np.uint64), s[f][rows].view(np.uint64)), (r, f)
        assert np.array_equal(got["state"]["bus_w"].view(np.uint64),
                              s["bus_w"][bus_owner == r].view(np.uint64)), r
        assert np.array_equal(got["state"]["branch_point"].view(np.uint64),
                              s["branch_point"].reshape(-1, 6)[br_owner == r].view(np.uint64)), r
