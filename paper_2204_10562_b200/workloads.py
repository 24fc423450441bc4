"""Deterministic synthetic planning workloads (BASELINE.json configs).

Every generator returns an :class:`InstanceSpec` — plain Python lists, no
package types — so the same inputs can be fed to the reference package (golden
generation, in the build container only), the C oracle (tests / CPU baseline)
and this package (``spec.to_model()``).

    C1  VGG-19 (19 layers) on a 4-GPU fully connected PCIe box, M = 8
    C2  BERT-large 24 layers on an 8-GPU DGX-1 hybrid cube-mesh, M = 32
    C3  GPT-style 96 layers on a 64-GPU 8x8 two-tier topology, M in 8..256
        (uniform and jittered variants)
    C4  4096 random 32-layer profiles x random heterogeneous 16-GPU cliques, M = 32
    C5  1024-layer chain on a 256-GPU random clique, M = 512, with the 256
        candidate plans xi = 1..256 (even split, contiguous devices)
"""

import math
import random
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

C3_MICROBATCHES = (8, 16, 32, 64, 128, 256)
C4_SEED = 20260822


@dataclass
class InstanceSpec:
    name: str
    fwd: List[float]
    bwd: List[float]
    param: List[float]
    efwd: List[float]
    ebwd: List[float]
    gpu_ids: List[int]
    links: List[Tuple[int, int, float]]
    M: int
    meta: dict = field(default_factory=dict)

    @property
    def L(self) -> int:
        return len(self.fwd)

    @property
    def V(self) -> int:
        return len(self.gpu_ids)

    def to_model(self):
        """(ModelProfile, ClusterGraph, M) of this package."""
        from .model import InterLayerEdge, LayerProfile, ModelProfile, make_cluster
        layers = tuple(LayerProfile(id=i + 1, fwd_time=f, bwd_time=b, param_bytes=p)
                       for i, (f, b, p) in enumerate(zip(self.fwd, self.bwd, self.param)))
        edges = tuple(InterLayerEdge(src=i + 1, dst=i + 2, fwd_bytes=a, bwd_bytes=b)
                      for i, (a, b) in enumerate(zip(self.efwd, self.ebwd)))
        profile = ModelProfile(name=self.name, microbatch_size=1, layers=layers, edges=edges)
        return profile, make_cluster(self.gpu_ids, self.links), self.M

    def with_m(self, M: int) -> "InstanceSpec":
        return InstanceSpec(self.name, self.fwd, self.bwd, self.param, self.efwd, self.ebwd,
                            self.gpu_ids, self.links, int(M), dict(self.meta))


def models_of(specs: Sequence["InstanceSpec"]):
    """(profile, cluster, M) triples where equal profiles / clusters are the SAME
    objects — how a user plans one physical cluster for several models and
    microbatch counts."""
    from .model import InterLayerEdge, LayerProfile, ModelProfile, make_cluster
    profiles, clusters, out = {}, {}, []
    for s in specs:
        pk = (s.name.split("_j")[0], tuple(s.fwd), tuple(s.bwd), tuple(s.param), tuple(s.efwd), tuple(s.ebwd))
        ck = (tuple(s.gpu_ids), tuple(s.links))
        if pk not in profiles:
            layers = tuple(LayerProfile(id=i + 1, fwd_time=f, bwd_time=b, param_bytes=p)
                           for i, (f, b, p) in enumerate(zip(s.fwd, s.bwd, s.param)))
            edges = tuple(InterLayerEdge(src=i + 1, dst=i + 2, fwd_bytes=a, bwd_bytes=b)
                          for i, (a, b) in enumerate(zip(s.efwd, s.ebwd)))
            profiles[pk] = ModelProfile(name=s.name, microbatch_size=1, layers=layers, edges=edges)
        if ck not in clusters:
            clusters[ck] = make_cluster(s.gpu_ids, s.links)
        out.append((profiles[pk], clusters[ck], s.M))
    return out


def _clique(ids: Sequence[int], bw_fn) -> List[Tuple[int, int, float]]:
    return [(a, b, float(bw_fn(a, b))) for i, a in enumerate(ids) for b in ids[i + 1:]]


# --------------------------------------------------------------------------- C1
_VGG_CONV = [  # (c_in, c_out, output side, pooled after)
    (3, 64, 224, False), (64, 64, 224, True),
    (64, 128, 112, False), (128, 128, 112, True),
    (128, 256, 56, False), (256, 256, 56, False), (256, 256, 56, False), (256, 256, 56, True),
    (256, 512, 28, False), (512, 512, 28, False), (512, 512, 28, False), (512, 512, 28, True),
    (512, 512, 14, False), (512, 512, 14, False), (512, 512, 14, False), (512, 512, 14, True),
]
_VGG_FC = [(25088, 4096), (4096, 4096), (4096, 1000)]


def c1_vgg19(M: int = 8, Z: int = 32, flops_per_s: float = 14e12) -> InstanceSpec:
    """VGG-19 at 224^2, microbatch Z = 32, 4 x V100 on 16 GB/s PCIe."""
    fwd, param, out_elems = [], [], []
    for cin, cout, s, pooled in _VGG_CONV:
        fwd.append(Z * (2.0 * 9 * cin * cout * s * s) / flops_per_s)
        param.append(4.0 * (9 * cin * cout + cout))
        side = s // 2 if pooled else s
        out_elems.append(cout * side * side)
    for cin, cout in _VGG_FC:
        fwd.append(Z * (2.0 * cin * cout) / flops_per_s)
        param.append(4.0 * (cin * cout + cout))
        out_elems.append(cout)
    bwd = [2.0 * f for f in fwd]
    edge = [4.0 * Z * e for e in out_elems[:-1]]
    ids = [1, 2, 3, 4]
    return InstanceSpec("c1_vgg19", fwd, bwd, param, list(edge), list(edge), ids,
                        _clique(ids, lambda a, b: 16e9), M)


# --------------------------------------------------------------------------- C2
_DGX1_FAST = {(1, 2), (3, 4), (5, 6), (7, 8), (1, 5), (2, 6), (3, 7), (4, 8)}
_DGX1_MID = {(1, 3), (2, 4), (5, 7), (6, 8), (1, 4), (2, 3), (5, 8), (6, 7)}


def c2_bert24(M: int = 32) -> InstanceSpec:
    L = 24
    eb = 4.0 * 6 * 512 * 1024
    ids = list(range(1, 9))

    def bw(a, b):
        return 50e9 if (a, b) in _DGX1_FAST else (25e9 if (a, b) in _DGX1_MID else 12e9)

    return InstanceSpec("c2_bert24", [0.010] * L, [0.020] * L, [4.0 * 12.6e6] * L,
                        [eb] * (L - 1), [eb] * (L - 1), ids, _clique(ids, bw), M)


# --------------------------------------------------------------------------- C3
def two_tier_cluster(nodes: int, per_node: int, intra: float = 450e9, inter: float = 12.5e9):
    ids = list(range(1, nodes * per_node + 1))
    return ids, _clique(ids, lambda a, b: intra if (a - 1) // per_node == (b - 1) // per_node else inter)


def c3_gpt96(M: int = 32, jitter_seed=None, nodes: int = 8, per_node: int = 8, L: int = 96) -> InstanceSpec:
    fwd = [0.004] * L
    bwd = [0.008] * L
    if jitter_seed is not None:
        rng = random.Random(jitter_seed)
        fwd, bwd = [], []
        for _ in range(L):
            fwd.append(0.004 * (1.0 + 0.05 * rng.uniform(-1.0, 1.0)))
            bwd.append(0.008 * (1.0 + 0.05 * rng.uniform(-1.0, 1.0)))
    eb = 2.0 * 4 * 2048 * 12288
    ids, links = two_tier_cluster(nodes, per_node)
    name = "c3_gpt96" + ("" if jitter_seed is None else f"_j{jitter_seed}")
    return InstanceSpec(name, fwd, bwd, [2.0 * 151e6] * L, [eb] * (L - 1), [eb] * (L - 1), ids, links, M,
                        {"jitter_seed": jitter_seed})


def c3_sweep(jitter_seeds=(None, 96)) -> List[InstanceSpec]:
    """The C3 planning batch: every M in 8..256 for each profile variant."""
    return [c3_gpt96(M, s) for s in jitter_seeds for M in C3_MICROBATCHES]


# --------------------------------------------------------------------------- C4
def _logu(rng: random.Random, lo: float, hi: float) -> float:
    return math.exp(rng.uniform(math.log(lo), math.log(hi)))


def random_chain(rng: random.Random, L: int):
    layers = [(_logu(rng, 1e-3, 1.0), _logu(rng, 1e-3, 2.0), _logu(rng, 1e6, 1e10)) for _ in range(L)]
    edges = [(_logu(rng, 1e5, 1e9), _logu(rng, 1e5, 1e9)) for _ in range(L - 1)]
    return ([a for a, _, _ in layers], [b for _, b, _ in layers], [c for _, _, c in layers],
            [a for a, _ in edges], [b for _, b in edges])


def c4_instance(k: int, L: int = 32, V: int = 16, M: int = 32) -> InstanceSpec:
    """conftest.random_instance's envelope (conftest.py:58-82) with L, V, M fixed."""
    rng = random.Random(C4_SEED + k)
    fwd, bwd, param, ef, eb = random_chain(rng, L)
    ids = list(range(1, V + 1))
    links = [(a, b, _logu(rng, 1e8, 1e11)) for i, a in enumerate(ids) for b in ids[i + 1:]]
    return InstanceSpec(f"c4_{k}", fwd, bwd, param, ef, eb, ids, links, M, {"k": k})


def c4_batch(n: int = 4096, start: int = 0) -> List[InstanceSpec]:
    return [c4_instance(k) for k in range(start, start + n)]


# --------------------------------------------------------------------------- C5
def c5_instance(L: int = 1024, V: int = 256, M: int = 512) -> InstanceSpec:
    fwd, bwd, param, ef, eb = random_chain(random.Random(1), L)
    rng = random.Random(2)
    ids = list(range(1, V + 1))
    links = [(a, b, _logu(rng, 1e8, 1e11)) for i, a in enumerate(ids) for b in ids[i + 1:]]
    return InstanceSpec("c5_chain1024", fwd, bwd, param, ef, eb, ids, links, M)


def even_split_plan(L: int, order: Sequence[int], n_stages: int):
    """Stages (layer_start, layer_end, devices) for an even layer split with the
    remainder to the front (baselines.py:41-48 rule) on contiguous slices of
    ``order``, again remainder to the front."""
    V = len(order)
    lb, lx = divmod(L, n_stages)
    db, dx = divmod(V, n_stages)
    out, ls, d0 = [], 1, 0
    for n in range(n_stages):
        nl = lb + (1 if n < lx else 0)
        nd = db + (1 if n < dx else 0)
        out.append((ls, ls + nl - 1, tuple(order[d0:d0 + nd])))
        ls += nl
        d0 += nd
    return out
