"""Bus-graph partition: host invariants (CPU), cross-rank
exchange-plan consistency over a 2-process gloo group (CPU), and on the GPU
bit-identity of partitioned solves with the single-part solve (the 1 vs k
parity test of SURVEY.md §4)."""
import os

import numpy as np
import pytest

from conftest import REPO, case_path

TO_ROWS = (2, 3, 6, 7)  # pji, qji, wj, thj


def plan(ex, part, p):
    """Python restatement of partition.cpp:make_plan (send/recv row lists)."""
    ng = len(ex["gen"])
    ends = ex["ends"]
    k = int(part.max()) + 1
    send = [[] for _ in range(k)]
    recv = [[] for _ in range(k)]
    for b, (f, t) in enumerate(ends):
        pf, pt = part[f], part[t]
        base = 2 * ng + 8 * b
        if pf == p and pt != p:
            send[pt] += [base + r for r in TO_ROWS]
        if pt == p and pf != p:
            recv[pf] += [base + r for r in TO_ROWS]
    return send, recv


@pytest.mark.parametrize("name,k", [("case118", 2), ("case118", 4), ("case30", 3)])
def test_partition_invariants(gridadmm, name, k):
    net = gridadmm.Network(case_path(name))
    part = net.partition(k)
    assert part.min() == 0 and part.max() == k - 1
    assert np.array_equal(part, net.partition(k))  # deterministic
    ex = net.export()
    # every row owned exactly once: gen rows by gen bus, branch rows by the side's bus
    owner = np.full(net.num_rows, -1)
    ng = len(ex["gen"])
    for g, row in enumerate(ex["gen"]):
        owner[2 * g] = owner[2 * g + 1] = part[int(row[0])]
    for b, (f, t) in enumerate(ex["ends"]):
        base = 2 * ng + 8 * b
        for r in (0, 1, 4, 5):
            owner[base + r] = part[f]
        for r in TO_ROWS:
            owner[base + r] = part[t]
    assert (owner >= 0).all()
    # send/recv lists agree pairwise
    plans = [plan(ex, part, p) for p in range(k)]
    for p in range(k):
        for q in range(k):
            assert plans[p][0][q] == plans[q][1][p]


def test_weighted_partition_balances_measured_cost(gridadmm):
    """gridadmm_network_set_branch_weights: the contiguous BFS cut balances
    1 per bus + (1 + w_b) per from-branch to within one bus's weight; NULL
    restores the class weights; negative weights are rejected."""
    net = gridadmm.Network(case_path("case118"))
    k = 3
    base = net.partition(k)
    ex = net.export()
    nl = net.num_branches
    w = (np.random.default_rng(3).pareto(1.2, nl) * 8).astype(np.int32)
    net.set_branch_weights(w)
    part = net.partition(k)
    assert np.array_equal(part, net.partition(k)) and not np.array_equal(part, base)
    bus_w = np.ones(net.num_buses, dtype=np.int64)
    for b, (f, _t) in enumerate(ex["ends"]):
        bus_w[f] += 1 + int(w[b])
    load = np.bincount(part, weights=bus_w, minlength=k)
    assert load.max() <= bus_w.sum() / k + bus_w.max()
    net.set_branch_weights(None)
    assert np.array_equal(net.partition(k), base)
    bad = w.copy()
    bad[5] = -1
    with pytest.raises(gridadmm.GridAdmmError) as e:
        net.set_branch_weights(bad)
    assert e.value.status == 3


def _rank_main(rank, world, path, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, REPO)
    import paper_2110_06879_b200 as ga
    net = ga.Network(path)
    part = net.partition(world)
    send, recv = plan(net.export(), part, rank)
    # each rank ships its send list to the peer, which checks it against its recv list
    gathered = [None] * world
    dist.all_gather_object(gathered, {"send": send, "recv": recv, "part": part.tolist()})
    ok = all(gathered[q]["part"] == gathered[0]["part"] for q in range(world))
    for q in range(world):
        if q != rank:
            ok = ok and gathered[q]["send"][rank] == recv[q] and gathered[q]["recv"][rank] == send[q]
    out[rank] = int(ok)
    dist.destroy_process_group()


def test_two_rank_gloo_plan_consistency(gridadmm):
    """The multi-process (NCCL) transport exchanges exactly these lists; two
    gloo ranks derive them independently and must agree (partition is a
    deterministic function of (case, k))."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_rank_main, args=(2, case_path("case118"), port, out), nprocs=2, join=True)
    assert out[0] == 1 and out[1] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("name,k", [("case118", 2), ("case118", 4), ("case30", 3), ("case9", 2)])
def test_partitioned_iterations_bit_identical(gridadmm, name, k):
    cfgs = []
    for parts in (1, k):
        cfg = gridadmm.Config("case118", eps=1e-5, partitions=parts)
        cfgs.append(cfg)
    net = gridadmm.Network(case_path(name))
    s1 = gridadmm.Session(net, cfgs[0])
    sk = gridadmm.Session(net, cfgs[1])
    r1, _ = s1.iterate(80)
    rk, _ = sk.iterate(80)
    assert r1.shape == rk.shape
    assert np.array_equal(r1.view(np.uint64), rk.view(np.uint64))
    a, b = s1.get_state(), sk.get_state()
    for f in a:
        assert np.array_equal(a[f].view(np.uint64), b[f].view(np.uint64)), f


@pytest.mark.gpu
def test_partition_by_measured_branch_costs_bit_identical(gridadmm):
    """Partition weighted by the TRON steps a first sweep measured
    (Session.branch_costs -> Network.set_branch_weights): the 3-part run
    stays bit-identical to one part."""
    net = gridadmm.Network(case_path("case118"))
    s1 = gridadmm.Session(net, gridadmm.Config("case118", eps=1e-5))
    s1.iterate(5)
    cost = np.asarray(s1.branch_costs(), dtype=np.int64)
    assert cost.shape == (net.num_branches,) and cost.max() > 0
    base = net.partition(3)
    net.set_branch_weights(np.minimum(cost, 1 << 20).astype(np.int32))
    assert not np.array_equal(net.partition(3), base)
    s1 = gridadmm.Session(net, gridadmm.Config("case118", eps=1e-5))
    s3 = gridadmm.Session(net, gridadmm.Config("case118", eps=1e-5, partitions=3))
    r1, _ = s1.iterate(60)
    r3, _ = s3.iterate(60)
    assert np.array_equal(r1.view(np.uint64), r3.view(np.uint64))
    a, b = s1.get_state(), s3.get_state()
    for f in a:
        assert np.array_equal(a[f].view(np.uint64), b[f].view(np.uint64)), f


@pytest.mark.gpu
def test_partitioned_full_solve_case9(gridadmm):
    net = gridadmm.Network(case_path("case9"))
    st1, r1 = gridadmm.solve(net, gridadmm.Config("case9", eps=1e-5))
    st3, r3 = gridadmm.solve(net, gridadmm.Config("case9", eps=1e-5, partitions=3))
    assert st1 == st3
    m1, m3 = r1.metrics(), r3.metrics()
    for key in m1:
        assert np.float64(m1[key]).view(np.uint64) == np.float64(m3[key]).view(np.uint64), key


@pytest.mark.gpu
def test_partitioned_synthetic_grid(gridadmm):
    from gridcases import synth
    path = synth.ensure_case("case2868rte", "/tmp/gridadmm_cases")
    net = gridadmm.Network(path)
    s1 = gridadmm.Session(net, gridadmm.Config("case_ACTIVSg70k"))
    s4 = gridadmm.Session(net, gridadmm.Config("case_ACTIVSg70k", partitions=4))
    r1, _ = s1.iterate(25)
    r4, _ = s4.iterate(25)
    assert np.array_equal(r1.view(np.uint64), r4.view(np.uint64))


@pytest.mark.gpu
def test_nccl_engine_single_rank_bit_identical(gridadmm):
    """The one-process-per-GPU engine (dist.cpp: NCCL loaded with dlopen, the
    norms all-reduced, the exchange plan of a 1-part partition) on this box's
    single GPU: same residual series and state as the plain session."""
    net = gridadmm.Network(case_path("case118"))
    cfg = gridadmm.Config("case118", eps=1e-5)
    s1 = gridadmm.Session(net, cfg)
    sd = gridadmm.Session.distributed(net, cfg, 0, 1, gridadmm.nccl_unique_id())
    r1, _ = s1.iterate(60)
    rd, _ = sd.iterate(60)
    assert np.array_equal(r1.view(np.uint64), rd.view(np.uint64))
    a, b = s1.get_state(), sd.get_state()
    for f in a:
        assert np.array_equal(a[f].view(np.uint64), b[f].view(np.uint64)), f
