"""Deterministic synthetic "-shaped" grids for the benchmark configs.

None of BASELINE.json's large cases (case2868rte, 9241/13659pegase,
ACTIVSg25k/70k) exist offline, so they are synthesized by
tiling the bundled MATPOWER cases (data/case30.m: rate-limited, 6-variable
branch NLPs; data/case118.m: unlimited, 4-variable) and connecting the tiles
with tie lines, then trimming/adding branches and generators so the bus,
generator and branch counts hit the published dimensions exactly
(SURVEY.md §8 table).  Construction (seeded, reproducible):

* tiles: case30 copies for ``limited_frac`` of the buses, case118 copies for
  the rest; bus ids renumbered; only the first tile keeps its REF bus, other
  REF buses become PV;
* per-tile jitter of r, x, b and cost coefficients by a factor in [0.95, 1.05];
* tie lines between consecutive tiles (a chain) plus random long-range ties,
  with parameters copied (jittered) from a random branch of the source tile;
  ties inherit the source tile's rate (0 for case118 tiles);
* exact bus count: leftover buses are radial PQ stubs;
* exact branch count: non-tree intra-tile branches (w.r.t. a BFS spanning
  tree of the base case) are dropped, or extra ties added;
* exact generator count: generators are dropped uniformly (each tile keeps at
  least one) or duplicated, then all loads are scaled so total demand is 55%
  of total generation capacity.

The output is MATPOWER text with shortest round-trip float formatting, so the
reference parser and ours read identical doubles.
"""
from __future__ import annotations

import os
import re
from typing import Dict, List

import numpy as np

DATA_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")

SHAPES = {  # (buses, generators, branches) — SURVEY.md §8 / PAPER.md:399-402
    "case2868rte": (2868, 600, 3808),
    "case9241pegase": (9241, 1445, 16049),
    "case13659pegase": (13659, 4092, 20467),
    "case_ACTIVSg25k": (25000, 4834, 32230),
    "case_ACTIVSg70k": (70000, 10390, 88207),
}


def _matrix(text: str, name: str) -> np.ndarray:
    text = "\n".join(line.split("%", 1)[0] for line in text.splitlines())
    m = re.search(r"mpc\." + name + r"\s*=\s*\[(.*?)\]", text, re.S)
    rows = [r.split() for r in m.group(1).split(";")]
    rows = [[float(v) for v in r] for r in rows if r]
    width = max(len(r) for r in rows)
    return np.array([r + [0.0] * (width - len(r)) for r in rows])


def load_base(name: str) -> Dict[str, np.ndarray]:
    with open(os.path.join(DATA_DIR, name + ".m")) as f:
        text = f.read()
    return {k: _matrix(text, k) for k in ("bus", "gen", "branch", "gencost")}


def _tree_edges(nbus_ids: np.ndarray, branch: np.ndarray) -> np.ndarray:
    """Mask of branches in a BFS spanning tree of the base case."""
    idx = {int(b): i for i, b in enumerate(nbus_ids)}
    adj: List[List[tuple]] = [[] for _ in nbus_ids]
    for k, (f, t) in enumerate(branch[:, :2].astype(int)):
        adj[idx[f]].append((idx[t], k))
        adj[idx[t]].append((idx[f], k))
    seen = np.zeros(len(nbus_ids), bool)
    tree = np.zeros(len(branch), bool)
    seen[0] = True
    q = [0]
    while q:
        u = q.pop(0)
        for v, k in adj[u]:
            if not seen[v]:
                seen[v] = True
                tree[k] = True
                q.append(v)
    return tree


def _fmt(v: float) -> str:
    if v == int(v) and abs(v) < 1e15:
        return str(int(v))
    return repr(float(v))


def generate(nbus: int, ngen: int, nbranch: int, limited_frac: float = 0.6, seed: int = 2110,
             name: str = "synthetic") -> str:
    """Returns MATPOWER text of a connected tiled grid with exactly
    (nbus, ngen, nbranch) in-service buses/generators/branches."""
    rng = np.random.default_rng(seed)
    bases = {"case30": load_base("case30"), "case118": load_base("case118")}
    for b in bases.values():
        b["tree"] = _tree_edges(b["bus"][:, 0], b["branch"])
    n30 = int(round(limited_frac * nbus / 30))
    n118 = max(0, (nbus - 30 * n30) // 118)
    while 30 * n30 + 118 * n118 > nbus:
        n30 -= 1
    kinds = ["case30"] * n30 + ["case118"] * n118
    order = rng.permutation(len(kinds))
    kinds = [kinds[i] for i in order]

    buses, gens, costs, branches = [], [], [], []
    tile_bus_ids: List[np.ndarray] = []
    tile_branch_src: List[int] = []  # tile index of each branch (-1 ties/stubs)
    tile_tree: List[bool] = []
    next_id = 1
    for t, kind in enumerate(kinds):
        b = bases[kind]
        ids = b["bus"][:, 0].astype(int)
        remap = {old: next_id + i for i, old in enumerate(ids)}
        next_id += len(ids)
        tile_bus_ids.append(np.array([remap[i] for i in ids]))
        for row in b["bus"]:
            r = row.copy()
            r[0] = remap[int(r[0])]
            if r[1] == 3 and t > 0:
                r[1] = 2
            buses.append(r)
        jit = lambda: rng.uniform(0.95, 1.05)
        for row, crow in zip(b["gen"], b["gencost"]):
            if row[7] == 0:
                continue
            r = row.copy()
            r[0] = remap[int(r[0])]
            gens.append(r)
            c = crow.copy()
            ncoef = int(c[3])
            c[4:4 + ncoef] *= jit()
            costs.append(c)
        for row, tr in zip(b["branch"], b["tree"]):
            if row[10] == 0:
                continue
            r = row.copy()
            r[0] = remap[int(r[0])]
            r[1] = remap[int(r[1])]
            r[2] *= jit()
            r[3] *= jit()
            r[4] *= jit()
            branches.append(r)
            tile_branch_src.append(t)
            tile_tree.append(bool(tr))

    def tie(t_from: int, t_to: int):
        src = bases[kinds[t_from]]["branch"]
        r = src[rng.integers(len(src))].copy()
        r[0] = rng.choice(tile_bus_ids[t_from])
        r[1] = rng.choice(tile_bus_ids[t_to])
        r[2] *= rng.uniform(0.95, 1.05)
        r[3] *= rng.uniform(0.95, 1.05)
        r[4] *= rng.uniform(0.95, 1.05)
        r[8] = 0.0  # plain line: no transformer tap / shift
        r[9] = 0.0
        if r[5] > 0:
            r[5] *= 2.0  # ties carry inter-area transfers
        branches.append(r)
        tile_branch_src.append(-1)
        tile_tree.append(True)

    # tiles on a 2-D lattice, two ties to the right and two to the lower
    # neighbour, plus random long-range ties (keeps the electrical diameter
    # ~2*sqrt(tiles) instead of a chain's ~tiles, so angles stay bounded)
    ntile = len(kinds)
    width = max(1, int(np.ceil(np.sqrt(ntile))))
    for t in range(ntile):
        r0, c0 = divmod(t, width)
        for nb in ((t + 1) if c0 + 1 < width and t + 1 < ntile else -1,
                   (t + width) if t + width < ntile else -1):
            if nb >= 0:
                tie(t, nb)
                tie(t, nb)
    for _ in range(ntile // 4):
        a, b2 = rng.integers(ntile, size=2)
        if a != b2:
            tie(int(a), int(b2))

    # radial PQ stubs for the exact bus count
    nstub = nbus - len(buses)
    for _ in range(nstub):
        host_tile = int(rng.integers(len(kinds)))
        host = int(rng.choice(tile_bus_ids[host_tile]))
        row = np.zeros_like(buses[0])
        row[:13] = [next_id, 1, rng.uniform(1, 10), rng.uniform(0, 3), 0, 0, 1, 1, 0, 135, 1,
                    1.05, 0.95]
        buses.append(row)
        src = bases[kinds[host_tile]]["branch"]
        r = src[rng.integers(len(src))].copy()
        r[0], r[1], r[8], r[9] = host, next_id, 0.0, 0.0
        branches.append(r)
        tile_branch_src.append(-1)
        tile_tree.append(True)
        next_id += 1

    # exact branch count: random long-range ties if short, else drop
    # non-tree intra-tile branches
    while len(branches) < nbranch:
        a, b2 = rng.integers(len(kinds), size=2)
        if a != b2:
            tie(int(a), int(b2))
    branches = np.array(branches)
    tile_tree = np.array(tile_tree)
    excess = len(branches) - nbranch
    if excess > 0:
        cand = np.nonzero(~tile_tree)[0]
        if excess > len(cand):
            raise ValueError("cannot trim enough branches for the requested shape")
        drop = rng.choice(cand, size=excess, replace=False)
        branches = np.delete(branches, drop, axis=0)
    # exact generator count
    gens = np.array(gens)
    costs = np.array(costs)
    if len(gens) > ngen:
        gen_tile = np.searchsorted(np.cumsum([len(x) for x in tile_bus_ids]), gens[:, 0] - 1,
                                   side="right")
        keep = np.zeros(len(gens), bool)
        first = {}
        for k, t in enumerate(gen_tile):  # one guaranteed generator per tile
            if t not in first:
                first[t] = k
                keep[k] = True
        rest = np.nonzero(~keep)[0]
        need = ngen - int(keep.sum())
        if need < 0:
            raise ValueError("too few generators for one per tile")
        keep[rng.choice(rest, size=need, replace=False)] = True
        gens, costs = gens[keep], costs[keep]
    elif len(gens) < ngen:
        add = rng.choice(len(gens), size=ngen - len(gens), replace=True)
        gens = np.vstack([gens, gens[add]])
        costs = np.vstack([costs, costs[add]])
    buses = np.array(buses)
    # scale each tile's demand to 55% of the generation left in that tile, so
    # tiles are near self-sufficient and tie flows stay small
    ends = np.cumsum([len(x) for x in tile_bus_ids])  # tile t owns ids (ends[t-1], ends[t]]
    bus_tile = np.searchsorted(ends, buses[:, 0] - 1, side="right")
    gen_tile = np.searchsorted(ends, gens[:, 0] - 1, side="right")
    cap = np.bincount(gen_tile, weights=gens[:, 8], minlength=ntile + 1)
    in_tile = bus_tile < ntile
    load = np.bincount(bus_tile[in_tile], weights=buses[in_tile, 2], minlength=ntile + 1)
    f = np.where(load > 0, 0.55 * cap / np.maximum(load, 1e-300), 1.0)
    buses[in_tile, 2] *= f[bus_tile[in_tile]]
    buses[in_tile, 3] *= f[bus_tile[in_tile]]

    out = [f"function mpc = {name}", "% synthetic tiled grid (paper_2110_06879_b200.synth)",
           "mpc.version = '2';", "mpc.baseMVA = 100;", "mpc.bus = ["]
    out += ["\t" + "\t".join(_fmt(v) for v in r[:13]) + ";" for r in buses]
    out += ["];", "mpc.gen = ["]
    out += ["\t" + "\t".join(_fmt(v) for v in r[:10]) + ";" for r in gens]
    out += ["];", "mpc.branch = ["]
    out += ["\t" + "\t".join(_fmt(v) for v in r[:13]) + ";" for r in branches]
    out += ["];", "mpc.gencost = ["]
    out += ["\t" + "\t".join(_fmt(v) for v in r[:4 + int(r[3])]) + ";" for r in costs]
    out += ["];", ""]
    return "\n".join(out)


def write_case(shape: str, path: str, seed: int = 2110, limited_frac: float = 0.6) -> str:
    nb, ng, nl = SHAPES[shape]
    text = generate(nb, ng, nl, limited_frac=limited_frac, seed=seed, name=shape + "_synth")
    with open(path, "w") as f:
        f.write(text)
    return path


def ensure_case(shape: str, directory: str, seed: int = 2110) -> str:
    """Writes (once) and returns the path of the synthetic case for `shape`."""
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, f"{shape}_synth_s{seed}.m")
    if not os.path.exists(path):
        write_case(shape, path + ".tmp", seed=seed)
        os.replace(path + ".tmp", path)
    return path
