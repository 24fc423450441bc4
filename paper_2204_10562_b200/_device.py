"""Host <-> device marshalling for the planning C-ABI.

Instances are packed with numpy into two flat host buffers (fp64 inputs and
int32 descriptors), moved with ONE pinned host-to-device copy each, and the
pp_batch descriptor is filled with raw device pointers (torch tensors are only
used as device allocations and for the current CUDA stream).  Outputs come
back with one device-to-host copy per dtype.
"""

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import threading

import numpy as np
import torch

from . import _lib
from ._lib import PPBatch, PPInstance, PPPlan, PPSimBatch

F64 = torch.float64
I32 = torch.int32


@dataclass
class Packed:
    """One instance as flat arrays (device indices = positions in sorted ids)."""
    ids: Sequence[int]
    fwd: np.ndarray
    bwd: np.ndarray
    param: np.ndarray
    efwd: np.ndarray   # length L (last entry unused)
    ebwd: np.ndarray
    bw: np.ndarray     # V x V

    @property
    def L(self):
        return int(self.fwd.shape[0])

    @property
    def V(self):
        return int(self.bw.shape[0])


def pack_profile(profile):
    """(fwd, bwd, param, efwd, ebwd) arrays of a profile (edge arrays padded to L)."""
    L = profile.num_layers
    fwd = np.fromiter((lp.fwd_time for lp in profile.layers), dtype=np.float64, count=L)
    bwd = np.fromiter((lp.bwd_time for lp in profile.layers), dtype=np.float64, count=L)
    par = np.fromiter((lp.param_bytes for lp in profile.layers), dtype=np.float64, count=L)
    efwd = np.zeros(L)
    ebwd = np.zeros(L)
    if L > 1:
        efwd[:L - 1] = [e.fwd_bytes for e in profile.edges]
        ebwd[:L - 1] = [e.bwd_bytes for e in profile.edges]
    return fwd, bwd, par, efwd, ebwd


def pack_cluster(cluster, arrays=None):
    """(sorted ids, dense V x V bandwidth matrix); `arrays` = bandwidth_arrays(cluster) if known."""
    ids = tuple(sorted(cluster.gpu_ids))
    V = len(ids)
    bw = np.zeros((V, V))
    if cluster.bandwidth:
        sid = np.array(ids)
        keys, vals = arrays if arrays is not None else bandwidth_arrays(cluster)
        ia, ib = np.searchsorted(sid, keys[:, 0]), np.searchsorted(sid, keys[:, 1])
        bw[ia, ib] = vals
        bw[ib, ia] = vals
    return ids, bw


def pack(profile, cluster) -> Packed:
    ids, bw = pack_cluster(cluster)
    return Packed(ids, *pack_profile(profile), bw)


def pack_clusters(clusters):
    """pack_cluster for many clusters at once, or None unless EVERY cluster is in
    the common valid form — each unordered pair once as an int key (a, b) with
    a < b, both GPUs known, bandwidth in [1e-100, 1e100] (what validate_cluster
    and check_cluster_range accept without a loop); callers then fall back to
    the per-cluster path, which raises the reference's first error.  One pass
    over all the bandwidth dicts, one sort and one searchsorted for the whole
    batch instead of a dozen numpy calls per cluster."""
    import itertools
    chain = itertools.chain.from_iterable
    n = len(clusters)
    Vs, Es = [], []
    for c in clusters:
        V = len(c.gpu_ids)
        if V == 0 or len(c.bandwidth) != V * (V - 1) // 2:
            return None
        Vs.append(V)
        Es.append(len(c.bandwidth))
    nv, ne = sum(Vs), sum(Es)
    try:
        ids_all = np.fromiter(chain(c.gpu_ids for c in clusters), dtype=np.int64, count=nv)
        keys = np.fromiter(chain(chain(c.bandwidth.keys() for c in clusters)), dtype=np.int64,
                           count=2 * ne).reshape(ne, 2)
        vals = np.fromiter(chain(c.bandwidth.values() for c in clusters), dtype=np.float64, count=ne)
    except (TypeError, ValueError, OverflowError):
        return None
    lim = 1 << 31
    if ((ids_all < -lim) | (ids_all >= lim)).any() or ((keys < -lim) | (keys >= lim)).any():
        return None
    Varr = np.asarray(Vs, dtype=np.int64)
    cv = np.repeat(np.arange(n, dtype=np.int64), Varr)
    ce = np.repeat(np.arange(n, dtype=np.int64), np.asarray(Es, dtype=np.int64))
    comb = np.sort((cv << 32) | (ids_all + lim))   # (cluster, id) sorted: each cluster's ids ascending
    if (np.diff(comb) == 0).any():
        return None
    a, b = keys[:, 0], keys[:, 1]
    if not (a < b).all() or not ((vals >= 1e-100) & (vals <= 1e100)).all():
        return None
    voff = np.concatenate(([0], np.cumsum(Varr)))
    sid_np = (comb & 0xffffffff) - lim
    # id -> position in its cluster's sorted ids: a dense table over each cluster's id
    # span when the spans are compact (the usual 0..V-1 / 1..V numbering), else a search
    lo_c, hi_c = sid_np[voff[:-1]], sid_np[voff[1:] - 1]
    span = hi_c - lo_c + 1
    if int(span.sum()) <= 8 * nv + 1024:
        soff = np.concatenate(([0], np.cumsum(span)))
        tab = np.full(int(soff[-1]), -1, dtype=np.int64)
        tab[np.repeat(soff[:-1] - lo_c, Varr) + sid_np] = np.arange(nv) - np.repeat(voff[:-1], Varr)
        lo_e, hi_e, so_e = lo_c[ce], hi_c[ce], soff[:-1][ce] - lo_c[ce]
        if ((a < lo_e) | (b > hi_e)).any():
            return None
        pa, pb = tab[so_e + a], tab[so_e + b]
        if ((pa < 0) | (pb < 0)).any():
            return None
    else:
        ka, kb = (ce << 32) | (a + lim), (ce << 32) | (b + lim)
        ia, ib = np.searchsorted(comb, ka), np.searchsorted(comb, kb)
        if ((ia >= nv) | (ib >= nv)).any() or not ((comb[np.minimum(ia, nv - 1)] == ka) &
                                                  (comb[np.minimum(ib, nv - 1)] == kb)).all():
            return None
        pa, pb = ia - voff[ce], ib - voff[ce]
    moff = np.concatenate(([0], np.cumsum(Varr * Varr)))
    Ve, mo = Varr[ce], moff[:-1][ce]
    flat = np.zeros(int(moff[-1]))
    flat[mo + pa * Ve + pb] = vals
    flat[mo + pb * Ve + pa] = vals
    sid = sid_np.tolist()
    return [(tuple(sid[voff[k]:voff[k + 1]]), flat[moff[k]:moff[k + 1]].reshape(Vs[k], Vs[k])) for k in range(n)]


def bandwidth_arrays(cluster):
    """(keys [n, 2] int64, values [n] float64) of cluster.bandwidth, in dict order."""
    import itertools
    bwd = cluster.bandwidth
    n = len(bwd)
    try:
        keys = np.fromiter(itertools.chain.from_iterable(bwd.keys()), dtype=np.int64, count=2 * n).reshape(n, 2)
    except (TypeError, ValueError):   # keys that are not int pairs: let the caller's checks report them
        keys = np.array(list(bwd.keys()))
    return keys, np.fromiter(bwd.values(), dtype=np.float64, count=n)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class _Staging:
    """Reusable pinned host buffers for the H2D copies (one per dtype).  Before
    a buffer is refilled, the event recorded after its previous copy is waited
    on, so an in-flight non_blocking copy is never overwritten."""

    def __init__(self):
        self.buf = {}
        self.evt = {}
        # fill + async copy + event record are one critical section: two threads
        # planning concurrently must not refill a buffer whose copy is queued
        self.lock = threading.Lock()

    def to_device(self, arr: np.ndarray, dev):
        with self.lock:
            return self._to_device(arr, dev)

    def _to_device(self, arr: np.ndarray, dev):
        key = arr.dtype.str
        n = arr.size
        buf = self.buf.get(key)
        if key in self.evt:
            self.evt[key].synchronize()
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(n, 1 << 16), dtype=torch.from_numpy(arr[:0]).dtype).pin_memory()
            self.buf[key] = buf
        view = buf[:n]
        view.numpy()[:] = arr.reshape(-1)
        out = view.to(dev, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.evt[key] = ev
        return out


_staging = _Staging()


def device():
    _lib.load(require_device=True)
    return torch.device("cuda", torch.cuda.current_device())


_INST_DTYPE = np.dtype([(name, np.int32 if t is C.c_int32 else np.int64) for name, t in PPInstance._fields_])
assert _INST_DTYPE.itemsize == C.sizeof(PPInstance)


class DeviceBatch:
    """A batch of planning instances resident on the GPU with all outputs.

    items: list of (Packed, M, flags, order_positions or None).
    workspace=False skips the pp_layout fp64 workspace (RDO / DP / sweep
    tables; L V^3 / 2 doubles at the largest shapes, 68 GB for 1024 x 256):
    such a batch serves pp_phi and caller-plan simulation (pp_simulate) only,
    and the library refuses the other entry points on it.
    """

    def __init__(self, items, capture_events=True, workspace=True):
        lib = _lib.load()
        dev = device()
        self.items = items
        n = len(items)
        self.n = n
        Ls = np.array([p.L for p, _, _, _ in items], dtype=np.int32)
        Vs = np.array([p.V for p, _, _, _ in items], dtype=np.int32)
        Ms = np.array([m for _, m, _, _ in items], dtype=np.int32)
        self.Ms = Ms.astype(np.int64)
        fl = np.array([f for _, _, f, _ in items], dtype=np.int32)
        inst = (PPInstance * n)()
        tot = [C.c_int64() for _ in range(8)]
        _lib.check(lib.pp_layout(n, Ls.ctypes.data, Vs.ctypes.data, Ms.ctypes.data, fl.ctypes.data,
                                 C.cast(inst, C.c_void_p), *[C.byref(t) for t in tot]))
        n_layer, n_bw, n_order, n_sweep, n_stage, n_ev, n_ar, n_ws = (t.value for t in tot)
        self.inst_host = inst
        self.sizes = dict(layer=n_layer, bw=n_bw, order=n_order, sweep=n_sweep, stage=n_stage,
                          ev=n_ev, ar=n_ar, ws=n_ws)
        # ---- fp64 input buffer: fwd | bwd | param | efwd | ebwd | bw
        fin = np.empty(5 * n_layer + n_bw)
        for k, (p, _, _, _) in enumerate(items):
            lo, L = inst[k].layer_off, p.L
            for s, arr in enumerate((p.fwd, p.bwd, p.param, p.efwd, p.ebwd)):
                fin[s * n_layer + lo: s * n_layer + lo + L] = arr
            fin[5 * n_layer + inst[k].bw_off: 5 * n_layer + inst[k].bw_off + p.V * p.V] = p.bw.reshape(-1)
        # ---- int32 buffer: instance descriptors (as raw int32 words) | order
        ib = np.frombuffer(bytes(inst), dtype=np.int32)
        order = np.zeros(n_order, dtype=np.int32)
        for k, (p, _, _, o) in enumerate(items):
            if o is not None:
                order[inst[k].order_off: inst[k].order_off + p.V] = o
        iin = np.concatenate([ib, order])
        self.max_L = int(Ls.max())
        self.max_V = int(Vs.max())
        # ---- device allocations
        self.d_fin = _staging.to_device(fin, dev)
        self.d_iin = _staging.to_device(iin, dev)
        # outputs: fp64 [sweep_w | sweep_mk | sweep_bound | best_mk | phi | gamma | ar_s | ar_e | ev_s | ev_e]
        ev = n_ev if capture_events else 0
        self.f_off = np.cumsum([0, n_sweep, n_sweep, n_sweep, n, n, n, n_ar, n_ar, ev, ev])
        self.d_fout = torch.empty(int(self.f_off[-1]), dtype=F64, device=dev)
        # int32 outputs: [sweep_r | ls | le | dlo | dhi | best_xi | ev_order]
        self.i_off = np.cumsum([0, n_sweep, n_stage, n_stage, n_stage, n_stage, n, ev])
        self.d_iout = torch.empty(int(self.i_off[-1]), dtype=I32, device=dev)
        self.d_ws = torch.empty(max(n_ws, 1), dtype=F64, device=dev) if workspace else None
        self.capture_events = capture_events
        self.n_ib = ib.size
        b = PPBatch()
        b.n_inst = n
        b.max_L = self.max_L
        b.max_V = self.max_V
        b.max_M = int(Ms.max())
        fp = self.d_fin.data_ptr()
        b.inst = self.d_iin.data_ptr()
        b.fwd = fp
        b.bwd = fp + 8 * n_layer
        b.param = fp + 16 * n_layer
        b.efwd = fp + 24 * n_layer
        b.ebwd = fp + 32 * n_layer
        b.bw = fp + 40 * n_layer
        b.order = self.d_iin.data_ptr() + 4 * ib.size
        fo = self.d_fout.data_ptr()
        fo_ = [fo + 8 * int(x) for x in self.f_off]
        b.sweep_w, b.sweep_mk, b.sweep_bound, b.best_mk, b.phi = fo_[0], fo_[1], fo_[2], fo_[3], fo_[4]
        b.gamma = fo_[5]
        b.ar_start, b.ar_end = fo_[6], fo_[7]
        b.ev_start = fo_[8] if capture_events else None
        b.ev_end = fo_[9] if capture_events else None
        io = self.d_iout.data_ptr()
        io_ = [io + 4 * int(x) for x in self.i_off]
        b.sweep_r, b.stage_ls, b.stage_le, b.stage_dlo, b.stage_dhi, b.best_xi = io_[:6]
        b.ev_order = io_[6] if capture_events else None
        b.ws = self.d_ws.data_ptr() if workspace else None
        self.batch = b
        self.lib = lib

    def inst_offsets(self):
        """Per-instance V and output offsets (order, sweep, stage, ar, ev) as int64 arrays."""
        if getattr(self, "_offs", None) is None:
            a = np.frombuffer(bytes(self.inst_host), dtype=_INST_DTYPE)
            self._offs = {"V": a["V"].astype(np.int64), "order": a["order_off"], "sweep": a["sweep_off"],
                          "stage": a["stage_off"], "ar": a["ar_off"], "ev": a["ev_off"]}
        return self._offs

    # -- launches -------------------------------------------------------------
    def run(self, what="spp"):
        fn = {"spp": self.lib.pp_spp, "rdo": self.lib.pp_rdo, "prm": self.lib.pp_prm,
              "phi": self.lib.pp_phi, "sweep": self.lib.pp_pe_sweep, "select": self.lib.pp_select}[what]
        _lib.check(fn(C.byref(self.batch), _stream()))

    # -- results --------------------------------------------------------------
    def fetch(self):
        """Copy the outputs to host numpy.  Everything but the schedule events in one
        D2H per dtype; the events (capacity M (4V - 3) per instance, of which the
        chosen plan uses M (4 xi - 3)) are then gathered on the device to just the
        used prefixes and copied compactly (h["ev_coff"][k] = instance k's offset)."""
        stream = torch.cuda.current_stream()
        fe, ie = int(self.f_off[8]), int(self.i_off[6])   # starts of ev_start / ev_order
        srcs = (self.d_fout[:fe], self.d_iout[:ie], self.d_iin[self.n_ib:])
        dst = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in srcs]
        for d, t in zip(dst, srcs):
            d.copy_(t, non_blocking=True)
        stream.synchronize()
        fo, io, order = (d.numpy() for d in dst)
        f = {k: fo[int(self.f_off[i]):int(self.f_off[i + 1])]
             for i, k in enumerate(("sweep_w", "sweep_mk", "sweep_bound", "best_mk", "phi", "gamma",
                                    "ar_start", "ar_end"))}
        g = {k: io[int(self.i_off[i]):int(self.i_off[i + 1])]
             for i, k in enumerate(("sweep_r", "ls", "le", "dlo", "dhi", "best_xi"))}
        f.update(g)
        f["order"] = order
        if self.capture_events:
            bx = g["best_xi"].astype(np.int64)
            ev_s = self.d_fout[fe:int(self.f_off[9])]
            ev_e = self.d_fout[int(self.f_off[9]):int(self.f_off[10])]
            ev_o = self.d_iout[ie:int(self.i_off[7])]
            # used prefix of instance k: M_k (4 xi_k - 3) events from its ev_off, gathered
            # on the device with one index (built there from n offsets / counts)
            cnt = np.where(bx > 0, self.Ms * (4 * bx - 3), 0)
            coff = np.concatenate(([0], np.cumsum(cnt)[:-1])).astype(np.int64)
            c = int(cnt.sum())
            self._d2h_events = c
            if c:
                dev = self.d_fout.device
                shift = torch.from_numpy(self.inst_offsets()["ev"] - coff).to(dev)
                idx = torch.repeat_interleave(shift, torch.from_numpy(cnt).to(dev), output_size=c)
                idx += torch.arange(c, device=dev)
                dev_f = torch.cat((ev_s.index_select(0, idx), ev_e.index_select(0, idx)))
                dev_i = ev_o.index_select(0, idx)
                hf = torch.empty(dev_f.shape, dtype=dev_f.dtype, pin_memory=True)
                hi = torch.empty(dev_i.shape, dtype=dev_i.dtype, pin_memory=True)
                hf.copy_(dev_f, non_blocking=True)
                hi.copy_(dev_i, non_blocking=True)
                stream.synchronize()
                hfn = hf.numpy()
                f["ev_start"], f["ev_end"], f["ev_order"] = hfn[:c], hfn[c:], hi.numpy()
            else:
                f["ev_start"] = f["ev_end"] = np.zeros(0)
                f["ev_order"] = np.zeros(0, np.int32)
            f["ev_coff"] = coff
        return f

    def d2h_bytes(self):
        """Bytes of the last fetch (events: only the chosen plans' prefixes)."""
        ev = getattr(self, "_d2h_events", None)
        if ev is None:   # before any fetch: the full capacity
            return (self.d_fout.numel() * 8 + self.d_iout.numel() * 4 + (self.d_iin.numel() - self.n_ib) * 4)
        return int(self.f_off[8]) * 8 + int(self.i_off[6]) * 4 + (self.d_iin.numel() - self.n_ib) * 4 + ev * 20

    def h2d_bytes(self):
        return self.d_fin.numel() * 8 + self.d_iin.numel() * 4

    def query(self, cells, max_xi):
        """PartitionSolver.solve cells: list of (inst, l, xi, r, i) (valid ranges)."""
        dev = self.d_fin.device
        q = np.asarray(cells, dtype=np.int32).reshape(-1, 5)
        nq = q.shape[0]
        d_q = torch.from_numpy(np.ascontiguousarray(q.T)).to(dev)
        w = torch.empty(nq, dtype=F64, device=dev)
        frag = torch.zeros(nq * 4 * max_xi, dtype=I32, device=dev)
        feas = torch.empty(nq, dtype=I32, device=dev)
        p = d_q.data_ptr()
        _lib.check(self.lib.pp_prm_query(C.byref(self.batch), nq, p, p + 4 * nq, p + 8 * nq, p + 12 * nq,
                                         p + 16 * nq, max_xi, w.data_ptr(), frag.data_ptr(), feas.data_ptr(),
                                         _stream()))
        return w.cpu().numpy(), frag.cpu().numpy().reshape(nq, max_xi, 4), feas.cpu().numpy()

    def min_cut(self, k, verts):
        dev = self.d_fin.device
        v = torch.tensor(list(verts), dtype=I32, device=dev)
        in_a = torch.zeros(len(verts), dtype=torch.uint8, device=dev)
        w = torch.empty(1, dtype=F64, device=dev)
        _lib.check(self.lib.pp_min_cut(C.byref(self.batch), k, v.data_ptr(), len(verts), in_a.data_ptr(),
                                       w.data_ptr(), _stream()))
        return in_a.cpu().numpy(), float(w.cpu().item())


@dataclass
class SimPlan:
    """A caller plan: stages (ls, le, device positions) + queues in chain order."""
    inst: int
    M: int
    stages: List[tuple]
    flags: int
    queues: Optional[List[List[tuple]]] = None   # per resource (chain order): [(m, pos), ...]


class SimRun:
    """Run pp_simulate for plans over a DeviceBatch's instances."""

    def __init__(self, db: DeviceBatch, plans: Sequence[SimPlan], capture_events=True, costs=False, launch=True):
        lib = db.lib
        dev = db.d_fin.device
        n = len(plans)
        P = (PPPlan * n)()
        ls, le, doff, devs, qoff, qitems = [], [], [], [], [], []
        lane = ev = ar = 0
        max_N = 1
        self.meta = []
        for k, sp in enumerate(plans):
            N = len(sp.stages)
            J = 4 * N - 3
            R = 2 * N - 1
            max_N = max(max_N, N)
            p = P[k]
            p.inst, p.N, p.M, p.flags = sp.inst, N, sp.M, sp.flags
            p.stage_off = len(ls)
            p.devoff_off = len(doff)
            for a, b_, d in sp.stages:
                ls.append(a); le.append(b_)
                doff.append(len(devs))
                devs.extend(d)
            doff.append(len(devs))
            p.queue_off = len(qoff)
            qbase = len(qitems) // 2
            if sp.queues is not None:
                cnt = 0
                for q in sp.queues:
                    qoff.append(qbase + cnt)
                    for m, pos in q:
                        qitems.extend((m, pos))
                    cnt += len(q)
                qoff.append(qbase + cnt)
            else:
                qoff.extend([qbase] * (R + 1))
            p.lane_off = lane; lane += R
            p.ev_off = ev; ev += sp.M * J
            p.ar_off = ar; ar += N
            self.meta.append((N, sp.M, J, R, p.lane_off, p.ev_off, p.ar_off))
        ib = np.frombuffer(bytes(P), dtype=np.int32)
        ints = [ib, np.array(ls, np.int32), np.array(le, np.int32), np.array(doff, np.int32),
                np.array(devs if devs else [0], np.int32), np.array(qoff, np.int32),
                np.array(qitems if qitems else [0, 0], np.int32)]
        offs = np.cumsum([0] + [a.size for a in ints])
        d_in = _staging.to_device(np.concatenate(ints), dev)
        # fp64 outputs: makespan | bound | ar_s | ar_e | ev_s | ev_e | scratch (generic queues only)
        #              | lane costs | workload (costs=True only)
        evn = ev if capture_events else 0
        scr = ev if any(sp.queues is not None for sp in plans) else 1
        nlc, nwl = (lane * _lib.PP_LANE_COST_FIELDS, n) if costs else (0, 0)
        self.f_off = np.cumsum([0, n, n, ar, ar, evn, evn, scr, nlc, nwl])
        self.d_f = torch.empty(int(self.f_off[-1]), dtype=F64, device=dev)
        # int32 outputs: status | head | cycles
        self.i_off = np.cumsum([0, n, lane, n])
        self.d_i = torch.empty(int(self.i_off[-1]), dtype=I32, device=dev)
        self.d_done = torch.empty(n, dtype=torch.int64, device=dev)
        s = PPSimBatch()
        s.n_plan, s.max_N = n, max_N
        ip = d_in.data_ptr()
        s.plan, s.ls, s.le, s.dev_off, s.devs, s.q_off, s.q_items = (ip + 4 * int(o) for o in offs[:7])
        fp = self.d_f.data_ptr()
        fo = [fp + 8 * int(x) for x in self.f_off]
        s.makespan, s.bound, s.ar_start, s.ar_end = fo[0], fo[1], fo[2], fo[3]
        s.ev_start = fo[4] if capture_events else None
        s.ev_end = fo[5] if capture_events else None
        s.scratch = fo[6]
        s.lane_cost = fo[7] if costs else None
        s.workload = fo[8] if costs else None
        io = self.d_i.data_ptr()
        s.status, s.head, s.cycles = io, io + 4 * n, io + 4 * int(self.i_off[2])
        s.n_done = self.d_done.data_ptr()
        self._keep = d_in
        self.sim = s
        self.n = n
        self.capture_events = capture_events
        self.costs = costs
        self.db = db
        if launch:
            self.launch()

    def launch(self):
        """(Re-)run pp_simulate over the uploaded plans on the current stream."""
        _lib.check(self.db.lib.pp_simulate(C.byref(self.db.batch), C.byref(self.sim), _stream()))

    def fetch(self):
        f = self.d_f.cpu().numpy()
        i = self.d_i.cpu().numpy()
        done = self.d_done.cpu().numpy()
        out = []
        for k, (N, M, J, R, lane, ev, ar) in enumerate(self.meta):
            rec = dict(makespan=float(f[self.f_off[0] + k]), bound=float(f[self.f_off[1] + k]),
                       status=int(i[k]), n_done=int(done[k]),
                       head=i[self.i_off[1] + lane: self.i_off[1] + lane + R],
                       ar_start=f[self.f_off[2] + ar: self.f_off[2] + ar + N],
                       ar_end=f[self.f_off[3] + ar: self.f_off[3] + ar + N])
            rec["cycles"] = int(i[self.i_off[2] + k])
            if self.capture_events:
                rec["ev_start"] = f[self.f_off[4] + ev: self.f_off[4] + ev + M * J]
                rec["ev_end"] = f[self.f_off[5] + ev: self.f_off[5] + ev + M * J]
            if self.costs:
                F_ = _lib.PP_LANE_COST_FIELDS
                rec["lane_cost"] = f[self.f_off[7] + lane * F_: self.f_off[7] + (lane + R) * F_].reshape(R, F_)
                rec["workload"] = float(f[self.f_off[8] + k])
            out.append(rec)
        return out
