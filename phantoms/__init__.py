"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no divergence, no label
update, no projection): it only draws phantoms and turns them into the data
terms D_L(x) and smoothness capacities S(x) that the paper's problem statement
takes as inputs (Eq. 1, Eq. 9).  The paper has no
datasets or experiments, so these phantoms stand in for its
medical-imaging motivation; the recipe is BASELINE.json's five
configs, with the unspecified details fixed in DESIGN.md §"Input recipe"
(SURVEY.md §8.4.1).

Determinism:
  * geometry and per-node constants come from a sequential SplitMix64 stream
    seeded with the config seed;
  * per-voxel Gaussian noise is counter based: Box-Muller on the SplitMix64
    outputs at positions 2i+1 and 2i+2 of a stream seeded with
    seed ^ 0x9E3779B97F4A7C15, where i is the GLOBAL linear voxel index
    (x fastest).  Any window of a volume is therefore generated identically
    to the same window cut from the whole volume.
  * intensities and D are computed in fp64 and rounded to fp32 (RNE); S is
    computed in fp64 from the fp32 intensity and rounded, subnormals flushed
    to zero.

Layouts returned (the C-ABI boundary layout): D is float32 [L][z][y][x]
(one volume per end label, x fastest); a shared S field is float32 [z][y][x].
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


# --------------------------------------------------------------------------
# SplitMix64
# --------------------------------------------------------------------------
def _mix_scalar(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


class SplitMix64:
    """Sequential SplitMix64 stream; uniform() = (x >> 11) * 2^-53."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        return _mix_scalar(self.state)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lo + (hi - lo) * ((self.next_u64() >> 11) * (1.0 / 9007199254740992.0))

    def randint(self, lo: int, hi: int) -> int:
        """Integer uniform on [lo, hi] (inclusive)."""
        return lo + min(int(self.uniform() * (hi - lo + 1)), hi - lo)


def _mix_array(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def gaussian_at(seed_noise: int, lin: np.ndarray) -> np.ndarray:
    """Standard normal deviates at global linear voxel indices `lin` (uint64)."""
    s = np.uint64(seed_noise & _MASK)
    lin = lin.astype(np.uint64)
    with np.errstate(over="ignore"):
        k1 = lin * np.uint64(2) + np.uint64(1)
        k2 = k1 + np.uint64(1)
        z1 = _mix_array(s + k1 * GOLDEN)
        z2 = _mix_array(s + k2 * GOLDEN)
    u1 = (z1 >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    u2 = (z2 >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    r = np.sqrt(-2.0 * np.log1p(-u1))  # 1 - u1 in (0, 1]
    return r * np.cos(2.0 * math.pi * u2)


# --------------------------------------------------------------------------
# Label graphs (node 0 = source S; edges (parent, child, w))
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Graph:
    num_nodes: int
    edges: List[Tuple[int, int, float]]
    names: List[str]

    @property
    def parent(self):
        return np.array([e[0] for e in self.edges], dtype=np.int32)

    @property
    def child(self):
        return np.array([e[1] for e in self.edges], dtype=np.int32)

    @property
    def weight(self):
        return np.array([e[2] for e in self.edges], dtype=np.float32)

    def leaves(self) -> List[int]:
        """End labels (childless non-source nodes) in node-id order."""
        has_child = {p for p, _, _ in self.edges}
        return [v for v in range(1, self.num_nodes) if v not in has_child]


def potts_graph(K: int) -> Graph:
    """Potts model as the star DAG S -> {L_0..L_{K-1}}, w = 1."""
    return Graph(K + 1, [(0, k + 1, 1.0) for k in range(K)], ["S"] + [f"L{k}" for k in range(K)])


def hmf_graph() -> Graph:
    """C3 hierarchy (reading R11): S->{A,B,C}; A->{L0,L1}; B->{L2,L3}; C->{L4,L5}."""
    e = [(0, 1, 1.0), (0, 2, 1.0), (0, 3, 1.0),
         (1, 4, 1.0), (1, 5, 1.0), (2, 6, 1.0), (2, 7, 1.0), (3, 8, 1.0), (3, 9, 1.0)]
    return Graph(10, e, ["S", "A", "B", "C", "L0", "L1", "L2", "L3", "L4", "L5"])


def dag_graph() -> Graph:
    """C4 DAG (reading R10): S->{A,B,C}; A->{L0,L1,L4:.5}; B->{L2,L3,L5:.5}; C->{L4:.5,L5:.5}."""
    e = [(0, 1, 1.0), (0, 2, 1.0), (0, 3, 1.0),
         (1, 4, 1.0), (1, 5, 1.0), (1, 8, 0.5),
         (2, 6, 1.0), (2, 7, 1.0), (2, 9, 0.5),
         (3, 8, 0.5), (3, 9, 0.5)]
    return Graph(10, e, ["S", "A", "B", "C", "L0", "L1", "L2", "L3", "L4", "L5"])


def ishikawa_graph(N: int) -> Graph:
    """Ishikawa model with N levels / N+1 ordered labels as a DAG chain: level nodes
    N_1..N_N (ids 1..N) with N_i -> N_{i+1}; end labels L_0..L_N (ids N+1..2N+1) with S -> L_0,
    S -> N_1, N_i -> L_i; all weights 1 (so W_(N_i, L_j) = 1 for j >= i: u_{N_i} = sum_{j>=i} u_j).
    Only the level nodes carry spatial flows; end labels get capacity 0."""
    e = [(0, N + 1, 1.0), (0, 1, 1.0)]
    for i in range(1, N + 1):
        e.append((i, N + 1 + i, 1.0))
        if i < N:
            e.append((i, i + 1, 1.0))
    names = ["S"] + [f"N{i}" for i in range(1, N + 1)] + [f"L{i}" for i in range(N + 1)]
    return Graph(2 * N + 2, e, names)


def wide_dag(ni: int, nl: int, seed: int) -> Graph:
    """A seeded random label DAG with `ni` internal nodes (ids 1..ni) and `nl` end labels (ids ni+1..ni+nl), for
    the graphs beyond the compiled kernel set (up to 31 non-source nodes, 16 end labels).  A random
    tree below S (internal node i hangs under S or an earlier internal node, weight 1; every internal node gets at
    least one end label), then about a quarter of the end labels and of the non-top internal nodes get a second,
    earlier parent with weights 0.5 / 0.5 -- so W_(S,L) = 1 stays exact for every end label (reading R9)."""
    rng = SplitMix64(seed)
    top = max(1, ni // 4)
    par = {}
    for i in range(1, ni + 1):
        par[i] = [(0, 1.0)] if i <= top else [(rng.randint(1, i - 1), 1.0)]
    has_child = {p for i in par for p, _ in par[i] if p != 0}
    bare = [i for i in range(1, ni + 1) if i not in has_child]
    assert len(bare) <= nl, "too few end labels for the internal tree"
    for k in range(nl):
        leaf = ni + 1 + k
        par[leaf] = [(bare[k], 1.0)] if k < len(bare) else [(rng.randint(0, ni), 1.0)]
    def second_parent(v, lo, hi):
        p0 = par[v][0][0]
        p1 = rng.randint(lo, hi)
        if p1 != p0:
            par[v] = [(p0, 0.5), (p1, 0.5)]
    for k in range(nl):
        if rng.uniform() < 0.25:
            second_parent(ni + 1 + k, 1, ni)
    for i in range(top + 1, ni + 1):
        if rng.uniform() < 0.25:
            second_parent(i, 1, i - 1)
    edges = sorted((p, v, w) for v in par for p, w in par[v])
    names = ["S"] + [f"N{i}" for i in range(1, ni + 1)] + [f"L{k}" for k in range(nl)]
    return Graph(ni + nl + 1, edges, names)


# --------------------------------------------------------------------------
# Configs (BASELINE.json configs[0..4]; unspecified details = SURVEY §8.4.1)
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Config:
    name: str
    ndim: int
    nx: int
    ny: int
    nz: int
    kind: str            # "potts" | "hmf" | "dag"
    classes: int         # number of intensity classes = number of end labels
    n_shapes: int        # discs (2D) or ellipsoids (3D)
    sigma: float
    dterm: str           # "abs" -> |I - mu|, "sq" -> (I - mu)^2
    s_kind: str          # "scalar" | "edge" | "per_node_uniform"
    s_value: float
    iters: int
    c: float = 0.25
    tau: float = 0.1
    cap: str = "l2"
    seed: int = 0
    wide_ni: int = 0     # kind "wide": internal nodes of wide_dag(wide_ni, classes, seed)

    @property
    def K(self) -> int:
        return self.classes

    @property
    def V(self) -> int:
        return self.nx * self.ny * self.nz

    def graph(self) -> Graph:
        if self.kind == "potts":
            return potts_graph(self.classes)
        if self.kind == "hmf":
            return hmf_graph()
        if self.kind == "dag":
            return dag_graph()
        if self.kind == "ishikawa":
            return ishikawa_graph(self.classes - 1)
        if self.kind == "wide":
            return wide_dag(self.wide_ni, self.classes, self.seed)
        raise ValueError(self.kind)

    def mu(self) -> np.ndarray:
        return np.arange(self.classes, dtype=np.float64) / (self.classes - 1)

    def resized(self, nx: int, ny: int, nz: int, name: Optional[str] = None) -> "Config":
        return dataclasses.replace(self, nx=nx, ny=ny, nz=nz, name=name or f"{self.name}@{nx}x{ny}x{nz}")


CONFIGS: Dict[str, Config] = {
    "C1": Config("C1", 2, 64, 64, 1, "potts", 3, 3, 0.20, "abs", "scalar", 0.1, 200, seed=1001),
    "C2": Config("C2", 3, 256, 256, 256, "potts", 8, 28, 0.15, "sq", "edge", 0.05, 300, seed=1002),
    "C3": Config("C3", 3, 256, 256, 256, "hmf", 6, 20, 0.15, "sq", "per_node_uniform", 0.0, 300, seed=1003),
    "C4": Config("C4", 3, 320, 320, 320, "dag", 6, 20, 0.15, "sq", "per_node_uniform", 0.0, 300, seed=1004),
    "C5": Config("C5", 3, 768, 768, 768, "potts", 16, 60, 0.15, "abs", "edge", 0.05, 200, seed=1005),
    # the Ishikawa model (Alg. 3) on C2's phantom -- 8 ordered labels = 7 levels
    "I2": Config("I2", 3, 256, 256, 256, "ishikawa", 8, 28, 0.15, "sq", "edge", 0.05, 300, seed=1002),
}


# --------------------------------------------------------------------------
# Phantom geometry
# --------------------------------------------------------------------------
def _geometry(cfg: Config):
    """Draw shapes (in voxel units) and per-node constants from the sequential stream."""
    rng = SplitMix64(cfg.seed)
    shapes = []
    if cfg.ndim == 2:
        n = float(min(cfg.nx, cfg.ny))
        for j in range(cfg.n_shapes):
            cx = rng.uniform(0.15, 0.85) * cfg.nx
            cy = rng.uniform(0.15, 0.85) * cfg.ny
            r = rng.uniform(0.08, 0.20) * n
            shapes.append(((cx, cy, 0.5), (r, r, float("inf")), 1 + (j % 2)))
    else:
        for _ in range(cfg.n_shapes):
            c = (rng.uniform(0.1, 0.9) * cfg.nx, rng.uniform(0.1, 0.9) * cfg.ny, rng.uniform(0.1, 0.9) * cfg.nz)
            a = (rng.uniform(0.05, 0.25) * cfg.nx, rng.uniform(0.05, 0.25) * cfg.ny, rng.uniform(0.05, 0.25) * cfg.nz)
            cls = rng.randint(1, cfg.classes - 1)
            shapes.append((c, a, cls))
    node_s = None
    if cfg.s_kind == "per_node_uniform":
        g = cfg.graph()
        node_s = np.zeros(g.num_nodes, dtype=np.float32)
        for v in range(1, g.num_nodes):
            node_s[v] = np.float32(rng.uniform(0.01, 0.2))
    return shapes, node_s


def _class_map(cfg: Config, shapes, z0, z1, y0, y1, x0, x1) -> np.ndarray:
    lab = np.zeros((z1 - z0, y1 - y0, x1 - x0), dtype=np.int32)
    for (c, a, cls) in shapes:
        lo, hi = [], []
        for ax, (s0, s1) in zip(range(3), ((x0, x1), (y0, y1), (z0, z1))):
            if math.isinf(a[ax]):
                lo.append(s0); hi.append(s1); continue
            l = max(s0, int(math.ceil(c[ax] - a[ax] - 0.5)))
            h = min(s1, int(math.floor(c[ax] + a[ax] - 0.5)) + 1)
            lo.append(l); hi.append(h)
        if any(h <= l for l, h in zip(lo, hi)):
            continue
        xs = (np.arange(lo[0], hi[0], dtype=np.float64) + 0.5 - c[0]) / a[0]
        ys = (np.arange(lo[1], hi[1], dtype=np.float64) + 0.5 - c[1]) / a[1]
        r2 = xs[None, None, :] ** 2 + ys[None, :, None] ** 2
        if not math.isinf(a[2]):
            zs = (np.arange(lo[2], hi[2], dtype=np.float64) + 0.5 - c[2]) / a[2]
            r2 = r2 + zs[:, None, None] ** 2
        inside = r2 <= 1.0
        sub = lab[lo[2] - z0:hi[2] - z0, lo[1] - y0:hi[1] - y0, lo[0] - x0:hi[0] - x0]
        np.copyto(sub, np.int32(cls), where=np.broadcast_to(inside, sub.shape))
    return lab


def _intensity32(cfg: Config, shapes, z0, z1, y0, y1, x0, x1) -> np.ndarray:
    lab = _class_map(cfg, shapes, z0, z1, y0, y1, x0, x1)
    mu = cfg.mu()
    zz, yy, xx = np.meshgrid(np.arange(z0, z1, dtype=np.uint64), np.arange(y0, y1, dtype=np.uint64),
                             np.arange(x0, x1, dtype=np.uint64), indexing="ij")
    lin = xx + np.uint64(cfg.nx) * (yy + np.uint64(cfg.ny) * zz)
    del xx, yy, zz
    noise = gaussian_at(cfg.seed ^ 0x9E3779B97F4A7C15, lin.ravel()).reshape(lin.shape)
    return (mu[lab] + cfg.sigma * noise).astype(np.float32)


def _flush_subnormal(a: np.ndarray) -> np.ndarray:
    tiny = np.finfo(np.float32).tiny
    a[np.abs(a) < tiny] = 0.0
    return a


@dataclasses.dataclass
class Inputs:
    cfg: Config
    graph: Graph
    window: Tuple[int, int, int, int, int, int]   # z0, z1, y0, y1, x0, x1 (global)
    D: np.ndarray                 # float32 [L][wz][wy][wx]
    s_kind: str                   # "scalar_per_node" | "shared_field"
    s_scalars: Optional[np.ndarray]   # float32 [num_nodes] (entry 0 ignored)
    s_field: Optional[np.ndarray]     # float32 [wz][wy][wx]
    intensity: np.ndarray         # float32 [wz][wy][wx]

    @property
    def shape(self):
        return self.D.shape[1:]

    def s_fields(self) -> List[np.ndarray]:
        """One capacity field per node id (index 0 = None), as float32 arrays (views where possible)."""
        out: List[Optional[np.ndarray]] = [None]
        leaves = set(self.graph.leaves())
        for v in range(1, self.graph.num_nodes):
            if self.cfg.kind == "ishikawa" and v in leaves:
                out.append(np.zeros(self.shape, dtype=np.float32))   # end labels carry no flow (Alg. 3)
            elif self.s_kind == "shared_field":
                out.append(self.s_field)
            else:
                out.append(np.full(self.shape, self.s_scalars[v], dtype=np.float32))
        return out


def generate(cfg: Config, window: Optional[Sequence[int]] = None) -> Inputs:
    """Generate D and S for `window` = (z0, z1, y0, y1, x0, x1) of the config's volume."""
    if window is None:
        window = (0, cfg.nz, 0, cfg.ny, 0, cfg.nx)
    z0, z1, y0, y1, x0, x1 = [int(v) for v in window]
    assert 0 <= z0 < z1 <= cfg.nz and 0 <= y0 < y1 <= cfg.ny and 0 <= x0 < x1 <= cfg.nx
    shapes, node_s = _geometry(cfg)
    g = cfg.graph()
    # extended by +1 (clipped) so forward differences of I are available for S
    ez1, ey1, ex1 = min(z1 + 1, cfg.nz), min(y1 + 1, cfg.ny), min(x1 + 1, cfg.nx)
    need_ext = cfg.s_kind == "edge"
    if need_ext:
        Iext = _intensity32(cfg, shapes, z0, ez1, y0, ey1, x0, ex1)
        I32 = Iext[: z1 - z0, : y1 - y0, : x1 - x0]
    else:
        I32 = _intensity32(cfg, shapes, z0, z1, y0, y1, x0, x1)
    I64 = I32.astype(np.float64)
    mu = cfg.mu()
    L = len(g.leaves())
    assert L == cfg.classes
    D = np.empty((L,) + I32.shape, dtype=np.float32)
    for l in range(L):
        if cfg.dterm == "abs":
            D[l] = np.abs(I64 - mu[l]).astype(np.float32)
        else:
            D[l] = ((I64 - mu[l]) ** 2).astype(np.float32)
    s_scalars = None
    s_field = None
    if cfg.s_kind == "scalar":
        s_kind = "scalar_per_node"
        s_scalars = np.full(g.num_nodes, cfg.s_value, dtype=np.float32)
        s_scalars[0] = 0.0
    elif cfg.s_kind == "per_node_uniform":
        s_kind = "scalar_per_node"
        s_scalars = node_s
    elif cfg.s_kind == "edge":
        s_kind = "shared_field"
        E = Iext.astype(np.float64)
        wz, wy, wx = I32.shape
        # forward differences of the noisy intensity, zero at the GLOBAL last index
        g2 = np.zeros(I32.shape, dtype=np.float64)
        m = min(wx, E.shape[2] - 1)
        g2[:, :, :m] += (E[:wz, :wy, 1:m + 1] - E[:wz, :wy, :m]) ** 2
        m = min(wy, E.shape[1] - 1)
        g2[:, :m, :] += (E[:wz, 1:m + 1, :wx] - E[:wz, :m, :wx]) ** 2
        if cfg.ndim == 3:
            m = min(wz, E.shape[0] - 1)
            g2[:m] += (E[1:m + 1, :wy, :wx] - E[:m, :wy, :wx]) ** 2
        s_field = _flush_subnormal((cfg.s_value * np.exp(-g2 / 0.01)).astype(np.float32))
    else:
        raise ValueError(cfg.s_kind)
    return Inputs(cfg, g, (z0, z1, y0, y1, x0, x1), D, s_kind, s_scalars, s_field, I32)


def config(name: str) -> Config:
    return CONFIGS[name]
