"""ctypes wrapper around oracle/liboracle.so.

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  Only tests/,
``__graft_entry__.smoke()`` (as the checker) and bench.py's CPU legs import
this module.  It exposes the C restatement of the reference planning path
(see the header of ``pipeplan_oracle.c`` for the file:line map) on plain
numpy arrays so it never depends on the product package.

An instance is described by the raw arrays the reference reads:
  fwd, bwd, param : float64[L]          (model.py:24-30)
  efwd, ebwd      : float64[L-1]        (model.py:33-39)
  bw              : float64[V, V]       symmetric, indexed by the position of
                                        the GPU id in sorted(gpu_ids)
  M               : microbatch count
Device indices everywhere are positions in sorted(gpu_ids).
"""

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

NEUMAIER = 1
NAIVE = 0


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class OrInst(C.Structure):
    _fields_ = [("L", C.c_int32), ("V", C.c_int32), ("M", C.c_int32), ("sum_mode", C.c_int32),
                ("fwd", C.c_void_p), ("bwd", C.c_void_p), ("param", C.c_void_p),
                ("efwd", C.c_void_p), ("ebwd", C.c_void_p), ("bw", C.c_void_p)]


class OrPlan(C.Structure):
    _fields_ = [("N", C.c_int32), ("ls", C.c_void_p), ("le", C.c_void_p),
                ("dev_off", C.c_void_p), ("devs", C.c_void_p), ("M", C.c_int32)]


class OrSimOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_done", C.c_int64),
                ("head_m", C.c_void_p), ("head_pos", C.c_void_p),
                ("n_events", C.c_int32),
                ("ev_start", C.c_void_p), ("ev_end", C.c_void_p),
                ("ev_m", C.c_void_p), ("ev_pos", C.c_void_p),
                ("n_ar", C.c_int32),
                ("ar_stage", C.c_void_p), ("ar_start", C.c_void_p), ("ar_end", C.c_void_p),
                ("makespan", C.c_double)]


class OrSppOut(C.Structure):
    _fields_ = [("order", C.c_void_p), ("feasible", C.c_void_p),
                ("workload", C.c_void_p), ("makespan", C.c_void_p), ("bound", C.c_void_p),
                ("best_xi", C.c_int32), ("frag", C.c_void_p),
                ("best_makespan", C.c_double), ("phi", C.c_double), ("theorem_factor", C.c_double),
                ("sim", OrSimOut)]


def _declare(L):
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.or_pysum.argtypes = [vp, i64, i32]; L.or_pysum.restype = dbl
    L.or_min_cut.argtypes = [vp, vp, i32, vp]; L.or_min_cut.restype = dbl
    L.or_rdo.argtypes = [vp, vp]; L.or_rdo.restype = None
    L.or_prm_new.argtypes = [vp, vp, i32]; L.or_prm_new.restype = vp
    L.or_prm_free.argtypes = [vp]; L.or_prm_free.restype = None
    L.or_prm_solve.argtypes = [vp, i32, i32, i32, i32, vp, vp]; L.or_prm_solve.restype = i32
    L.or_prm_best.argtypes = [vp, i32, vp, vp]; L.or_prm_best.restype = i32
    L.or_prm_W.argtypes = [vp, i32, i32, i32, i32]; L.or_prm_W.restype = dbl
    L.or_prm_feasible.argtypes = [vp, i32, i32, i32, i32]; L.or_prm_feasible.restype = i32
    L.or_pe_queues.argtypes = [i32, i32, vp, vp]; L.or_pe_queues.restype = None
    L.or_simulate.argtypes = [vp, vp, vp, vp, i32, vp]; L.or_simulate.restype = i32
    L.or_lemma1_bound.argtypes = [vp, vp]; L.or_lemma1_bound.restype = dbl
    L.or_phi.argtypes = [vp]; L.or_phi.restype = dbl
    L.or_spp.argtypes = [vp, vp]; L.or_spp.restype = i32
    L.or_spp_batch.argtypes = [i32, vp, vp, vp, i32]; L.or_spp_batch.restype = i32
    L.or_simulate_pe_batch.argtypes = [vp, i32, vp, vp, i32]; L.or_simulate_pe_batch.restype = i32


def _p(a):
    return a.ctypes.data


class Instance:
    """Owns contiguous arrays and the C struct pointing into them."""

    def __init__(self, fwd, bwd, param, efwd, ebwd, bw, M, sum_mode=NEUMAIER):
        self.fwd = np.ascontiguousarray(fwd, dtype=np.float64)
        self.bwd = np.ascontiguousarray(bwd, dtype=np.float64)
        self.param = np.ascontiguousarray(param, dtype=np.float64)
        self.efwd = np.ascontiguousarray(efwd, dtype=np.float64).reshape(-1)
        self.ebwd = np.ascontiguousarray(ebwd, dtype=np.float64).reshape(-1)
        self.bw = np.ascontiguousarray(bw, dtype=np.float64)
        self.L = int(self.fwd.shape[0])
        self.V = int(self.bw.shape[0])
        self.M = int(M)
        # keep a non-empty buffer for L == 1 (no edges)
        if self.efwd.size == 0:
            self.efwd = np.zeros(1); self.ebwd = np.zeros(1)
        self.c = OrInst(self.L, self.V, self.M, int(sum_mode), _p(self.fwd), _p(self.bwd), _p(self.param),
                        _p(self.efwd), _p(self.ebwd), _p(self.bw))

    def ref(self):
        return C.byref(self.c)


def pysum(x, mode=NEUMAIER):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().or_pysum(_p(x), x.size, mode)


def min_cut(inst, verts):
    verts = np.ascontiguousarray(sorted(verts), dtype=np.int32)
    in_a = np.zeros(verts.size, dtype=np.uint8)
    w = lib().or_min_cut(inst.ref(), _p(verts), verts.size, _p(in_a))
    a = tuple(int(v) for v, f in zip(verts, in_a) if f)
    b = tuple(int(v) for v, f in zip(verts, in_a) if not f)
    return a, b, w


def rdo(inst):
    order = np.zeros(inst.V, dtype=np.int32)
    lib().or_rdo(inst.ref(), _p(order))
    return tuple(int(v) for v in order)


class Prm:
    """Full DP table for one (instance, order, allow_replication)."""

    def __init__(self, inst, order, allow_replication=True):
        self.inst = inst
        self.order = np.ascontiguousarray(order, dtype=np.int32)
        self.h = lib().or_prm_new(inst.ref(), _p(self.order), int(bool(allow_replication)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_prm_free(self.h)
            self.h = None

    def _frags(self, n):
        return np.zeros(4 * max(n, 1), dtype=np.int32)

    def solve(self, l, xi, r, i):
        """(status, w, fragments) with fragments (ls, le, (dev ranks...))."""
        w = C.c_double(0.0)
        fr = self._frags(xi)
        st = lib().or_prm_solve(self.h, l, xi, r, i, C.byref(w), _p(fr))
        return st, w.value, (self._to_frags(fr, xi) if st == 1 else None)

    def best(self, xi):
        w = C.c_double(0.0)
        fr = self._frags(xi)
        st = lib().or_prm_best(self.h, xi, C.byref(w), _p(fr))
        return st, w.value, (self._to_frags(fr, xi) if st == 1 else None)

    def W(self, l, xi, r, i):
        return lib().or_prm_W(self.h, l, xi, r, i)

    def feasible(self, l, xi, r, i):
        return bool(lib().or_prm_feasible(self.h, l, xi, r, i))

    def _to_frags(self, fr, xi):
        out = []
        for n in range(xi):
            ls, le, lo, hi = (int(v) for v in fr[4 * n:4 * n + 4])
            out.append((ls, le, tuple(int(self.order[d - 1]) for d in range(lo, hi + 1))))
        return tuple(out)


def pe_queues(N, M):
    J = 4 * N - 3
    q_off = np.zeros(2 * N, dtype=np.int32)
    items = np.zeros(2 * M * J, dtype=np.int32)
    lib().or_pe_queues(N, M, _p(q_off), _p(items))
    return q_off, items.reshape(-1, 2)


class Plan:
    """stages: sequence of (layer_start, layer_end, device-index tuple)."""

    def __init__(self, stages, M):
        self.N = len(stages)
        self.M = int(M)
        self.ls = np.array([s[0] for s in stages], dtype=np.int32)
        self.le = np.array([s[1] for s in stages], dtype=np.int32)
        offs = [0]
        devs = []
        for s in stages:
            devs.extend(s[2]); offs.append(len(devs))
        self.dev_off = np.array(offs, dtype=np.int32)
        self.devs = np.array(devs if devs else [0], dtype=np.int32)
        self.c = OrPlan(self.N, _p(self.ls), _p(self.le), _p(self.dev_off), _p(self.devs), self.M)


def _sim_out(N, M):
    J = 4 * N - 3
    cap = max(M * J, 1)
    bufs = dict(head_m=np.zeros(2 * N, np.int32), head_pos=np.zeros(2 * N, np.int32),
                ev_start=np.zeros(cap), ev_end=np.zeros(cap),
                ev_m=np.zeros(cap, np.int32), ev_pos=np.zeros(cap, np.int32),
                ar_stage=np.zeros(N, np.int32), ar_start=np.zeros(N), ar_end=np.zeros(N))
    o = OrSimOut()
    for k, v in bufs.items():
        setattr(o, k, _p(v))
    return o, bufs


def simulate(inst, plan, q_off=None, items=None, forward_barrier=False):
    """Returns dict(status, n_done, heads, events[(m,pos,start,end)], ar[(s,start,end)], makespan)."""
    if q_off is None:
        q_off, items = pe_queues(plan.N, plan.M)
    q_off = np.ascontiguousarray(q_off, dtype=np.int32)
    items = np.ascontiguousarray(items, dtype=np.int32).reshape(-1)
    if items.size == 0:
        items = np.zeros(2, np.int32)
    o, b = _sim_out(plan.N, plan.M)
    st = lib().or_simulate(inst.ref(), C.byref(plan.c), _p(q_off), _p(items), int(bool(forward_barrier)), C.byref(o))
    R = 2 * plan.N - 1
    res = dict(status=st, n_done=o.n_done, makespan=o.makespan)
    if st == 0:
        n = o.n_events
        res["events"] = list(zip(b["ev_m"][:n].tolist(), b["ev_pos"][:n].tolist(),
                                 b["ev_start"][:n].tolist(), b["ev_end"][:n].tolist()))
        res["ar"] = list(zip(b["ar_stage"][:o.n_ar].tolist(), b["ar_start"][:o.n_ar].tolist(),
                             b["ar_end"][:o.n_ar].tolist()))
    else:
        res["heads"] = list(zip(b["head_m"][:R].tolist(), b["head_pos"][:R].tolist()))
    return res


def lemma1_bound(inst, plan):
    return lib().or_lemma1_bound(inst.ref(), C.byref(plan.c))


def phi(inst):
    return lib().or_phi(inst.ref())


def spp(inst, with_events=True):
    V, M = inst.V, inst.M
    cap = M * (4 * V - 3)
    bufs = dict(order=np.zeros(V, np.int32), feasible=np.zeros(V, np.uint8), workload=np.zeros(V),
                makespan=np.zeros(V), bound=np.zeros(V), frag=np.zeros(4 * V, np.int32))
    o = OrSppOut()
    for k, v in bufs.items():
        setattr(o, k, _p(v))
    sb = {}
    if with_events:
        o.sim, sb = _sim_out(V, M)
    best = lib().or_spp(inst.ref(), C.byref(o))
    order = tuple(int(v) for v in bufs["order"])
    frags = []
    for n in range(best):
        ls, le, lo, hi = (int(v) for v in bufs["frag"][4 * n:4 * n + 4])
        frags.append((ls, le, tuple(order[d - 1] for d in range(lo, hi + 1))))
    res = dict(order=order, best_xi=best, frags=tuple(frags), makespan=o.best_makespan,
               phi=o.phi, theorem_factor=o.theorem_factor,
               sweep=[(xi + 1, bool(bufs["feasible"][xi]), float(bufs["workload"][xi]),
                       float(bufs["makespan"][xi]) if bufs["feasible"][xi] else None,
                       float(bufs["bound"][xi]) if bufs["feasible"][xi] else None) for xi in range(V)])
    if with_events:
        n = o.sim.n_events
        res["events"] = list(zip(sb["ev_m"][:n].tolist(), sb["ev_pos"][:n].tolist(),
                                 sb["ev_start"][:n].tolist(), sb["ev_end"][:n].tolist()))
        res["ar"] = list(zip(sb["ar_stage"][:o.sim.n_ar].tolist(), sb["ar_start"][:o.sim.n_ar].tolist(),
                             sb["ar_end"][:o.sim.n_ar].tolist()))
    return res


def spp_batch(insts, nthreads):
    arr = (OrInst * len(insts))(*[i.c for i in insts])
    mk = np.zeros(len(insts))
    bx = np.zeros(len(insts), np.int32)
    lib().or_spp_batch(len(insts), arr, _p(mk), _p(bx), int(nthreads))
    return mk, bx


def simulate_pe_batch(inst, plans, nthreads):
    arr = (OrPlan * len(plans))(*[p.c for p in plans])
    mk = np.zeros(len(plans))
    lib().or_simulate_pe_batch(inst.ref(), len(plans), arr, _p(mk), int(nthreads))
    return mk
