"""validate_schedule (reference scheduler.py:303-452) on the GPU.

The host does what is inherently string work: it maps every event's block
label to its index in the plan's expected-block list and compares its
resource string, then formats the violation messages.  Every check — slot
occupancy and duplicates, durations against the device cost pass, the six
per-(microbatch, channel) ordering rules, AllReduce windows, per-resource
overlap (bitonic sort per resource), the barrier and the makespan — runs in
csrc/validate.cu (pp_validate_schedule), in two launches: the structural
phase, and the ordering phase only when the structure is sound (the
reference returns early the same way, scheduler.py:357-359).
"""

import ctypes as C
from typing import Dict, List

import numpy as np
import torch

from . import _device, _lib
from .cost import _check_costed_plan, _plan_costs
from .model import BWD, COMM_BWD, COMM_FWD, FWD, FWDBWD, ClusterGraph, LazyEvents, ModelProfile, Plan, Schedule, \
    ValidationError

_VAL_SORT_MAX = 8192


class PPValidateArgs(C.Structure):
    _fields_ = [("N", C.c_int32), ("M", C.c_int32), ("flags", C.c_int32), ("n_exp", C.c_int32),
                ("n_ev", C.c_int64),
                ("ev_m", C.c_void_p), ("ev_e", C.c_void_p), ("ev_res_ok", C.c_void_p),
                ("ev_start", C.c_void_p), ("ev_end", C.c_void_p), ("lane_cost", C.c_void_p),
                ("win_has", C.c_void_p), ("win_start", C.c_void_p), ("win_end", C.c_void_p),
                ("n_win_all", C.c_int32), ("win_all_end", C.c_void_p), ("makespan", C.c_double),
                ("slot_first", C.c_void_p), ("slot_last", C.c_void_p), ("slot_count", C.c_void_p),
                ("ev_flags", C.c_void_p), ("slot_flags", C.c_void_p), ("mn_flags", C.c_void_p),
                ("ar_flags", C.c_void_p), ("ov_flags", C.c_void_p), ("ov_idx", C.c_void_p),
                ("res_off", C.c_void_p), ("part", C.c_void_p), ("scal", C.c_void_p), ("stat", C.c_void_p),
                ("sort_ks", C.c_void_p), ("sort_ke", C.c_void_p), ("sort_ki", C.c_void_p), ("sort_cap", C.c_int64)]


def _expected(N: int, merged: bool):
    """[(label, resource, lane, field)] in the reference's expected order (scheduler.py:325-338)."""
    out = []
    for n in range(1, N + 1):
        if n == N and merged:
            out.append((f"{FWDBWD}{N}", f"stage{n}"))
        else:
            out.append((f"{FWD}{n}", f"stage{n}"))
            out.append((f"{BWD}{n}", f"stage{n}"))
    for n in range(1, N):
        out.append((f"{COMM_FWD}{n}", f"chan{n}"))
        out.append((f"{COMM_BWD}{n}", f"chan{n}"))
    return out


def _expected_duration(lc, N, merged, e, S):
    """The lane record field the kernel compares index e against (ValLayout::dur)."""
    if e < S:
        n = e // 2 + 1
        row = lc[2 * (n - 1)]
        if merged and n == N:
            return float(row[0])
        return float(row[5] if e & 1 else row[4])
    n = (e - S) // 2 + 1
    row = lc[2 * n - 1]
    return float(row[1] if (e - S) & 1 else row[0])


class _Events:
    """Event columns + accessors for messages, from LazyEvents or any sequence."""

    def __init__(self, events):
        if isinstance(events, LazyEvents):
            self.lazy = events
            em, ep, es, ee = events._arrays()
            self.m = np.ascontiguousarray(em, np.int32)
            self.start = np.ascontiguousarray(es, np.float64)
            self.end = np.ascontiguousarray(ee, np.float64)
            self.res_names, self.lab_names = events._res, events._lab
            self.q = np.asarray(ep, np.int64)
        else:
            self.lazy = None
            self.objs = tuple(events)
            self.m = np.array([e.microbatch for e in self.objs], np.int64)
            self.start = np.array([e.start for e in self.objs], np.float64)
            self.end = np.array([e.end for e in self.objs], np.float64)

    def __len__(self):
        return len(self.m)

    def labels(self):
        if self.lazy is not None:
            return {self.lab_names[q] for q in np.unique(self.q).tolist()}
        return {e.block for e in self.objs}

    def block(self, k):
        return self.lab_names[int(self.q[k])] if self.lazy is not None else self.objs[k].block

    def resource(self, k):
        return self.res_names[int(self.q[k])] if self.lazy is not None else self.objs[k].resource

    def micro(self, k):
        return int(self.m[k]) if self.lazy is not None else self.objs[k].microbatch

    def encode(self, index: Dict[str, int], exp_res: List[str]):
        """(expected index, resource matches) per event."""
        if self.lazy is not None:
            nq = len(self.lab_names)
            e_of = np.array([index.get(self.lab_names[q], -1) if self.lab_names[q] is not None else -1
                             for q in range(nq)], np.int32)
            ok_of = np.array([e_of[q] >= 0 and self.res_names[q] == exp_res[e_of[q]] for q in range(nq)], np.uint8)
            return e_of[self.q], ok_of[self.q]
        e = np.array([index.get(ev.block, -1) for ev in self.objs], np.int32)
        ok = np.array([x >= 0 and ev.resource == exp_res[x] for x, ev in zip(e.tolist(), self.objs)], np.uint8)
        return e, ok


def validate_schedule(schedule: Schedule, plan: Plan, profile: ModelProfile, cluster: ClusterGraph,
                      forward_barrier: bool = False) -> List[str]:
    """Every dependency / resource violation as a message, [] when valid (scheduler.py:303-452)."""
    N, M = plan.num_stages, plan.microbatch_count
    for k, s in enumerate(plan.stages, start=1):
        if s.index != k:
            raise ValidationError(f"stage at position {k} carries index {s.index}")
    _check_costed_plan(plan, profile, cluster)
    rec = _plan_costs([[(s.layer_start, s.layer_end, list(s.devices)) for s in plan.stages]], profile, cluster, M=M)[0]
    lc = np.ascontiguousarray(rec["lane_cost"])
    ev = _Events(schedule.events)
    E = len(ev)
    merged = f"{FWDBWD}{N}" in ev.labels()
    exp = _expected(N, merged)
    n_exp = len(exp)
    S = 2 * N - (1 if merged else 0)
    index = {lab: k for k, (lab, _) in enumerate(exp)}
    exp_res = [r for _, r in exp]
    e_code, res_ok = ev.encode(index, exp_res)
    ev_m = np.clip(ev.m, -2 ** 31, 2 ** 31 - 1).astype(np.int32)

    windows = {}
    for w in schedule.allreduce:
        windows[w.stage] = w
    win_has = np.array([1 if n in windows else 0 for n in range(1, N + 1)], np.uint8)
    win_s = np.array([windows[n].start if n in windows else 0.0 for n in range(1, N + 1)], np.float64)
    win_e = np.array([windows[n].end if n in windows else 0.0 for n in range(1, N + 1)], np.float64)
    win_all = np.array([w.end for w in schedule.allreduce] or [0.0], np.float64)

    dev = _device.device()
    lib = _lib.load()
    n_slot = M * n_exp
    i32 = lambda n: torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    u8 = lambda n: torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    f64 = lambda n: torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a) if a.size else np.zeros(1, a.dtype)).to(dev)
    t_m, t_e, t_ok, t_s, t_t = to(ev_m), to(e_code), to(res_ok), to(ev.start), to(ev.end)
    t_lc, t_wh, t_ws, t_we, t_wa = to(lc.reshape(-1)), to(win_has), to(win_s), to(win_e), to(win_all)
    # per-resource blocks of ov_idx: stage n hosts 2 labels (1 when merged last), chan n 2
    per_lane = [(1 if (r % 2 == 0 and r // 2 + 1 == N and merged) else 2) * M for r in range(2 * N - 1)]
    res_off = np.concatenate([[0], np.cumsum(per_lane)]).astype(np.int32)
    t_ro = to(res_off)
    out = dict(slot_first=i32(n_slot), slot_last=i32(n_slot), slot_count=i32(n_slot), ev_flags=u8(E),
               slot_flags=u8(n_slot), mn_flags=u8(M * N), ar_flags=u8(N), ov_flags=u8(n_slot), ov_idx=i32(n_slot),
               part=f64(3 * M + N), scal=f64(4), stat=i32(3))
    a = PPValidateArgs()
    a.N, a.M, a.flags, a.n_exp, a.n_ev = N, M, (1 if merged else 0) | (2 if forward_barrier else 0), n_exp, E
    a.ev_m, a.ev_e, a.ev_res_ok, a.ev_start, a.ev_end = (t.data_ptr() for t in (t_m, t_e, t_ok, t_s, t_t))
    a.lane_cost, a.win_has, a.win_start, a.win_end = (t.data_ptr() for t in (t_lc, t_wh, t_ws, t_we))
    a.n_win_all, a.win_all_end, a.makespan = len(schedule.allreduce), t_wa.data_ptr(), float(schedule.makespan)
    for k, t in out.items():
        setattr(a, k, t.data_ptr())
    a.res_off = t_ro.data_ptr()
    stream = _device._stream()
    _lib.check(lib.pp_validate_schedule(C.byref(a), 1, stream))

    # ---------------- phase 1 messages (scheduler.py:316-359)
    problems: List[str] = []
    evf = out["ev_flags"].cpu().numpy()[:E]
    # duplicates among events the slots do not cover (unknown block / microbatch): host dict
    loose = np.nonzero(evf & 12)[0]
    if loose.size:
        seen = set()
        for k in loose.tolist():
            key = (ev.micro(k), ev.block(k))
            if key in seen:
                evf[k] |= 1
            seen.add(key)
    for k in np.nonzero(evf & 3)[0].tolist():
        if evf[k] & 1:
            problems.append(f"duplicate event for microbatch {ev.micro(k)} block {ev.block(k)}")
        if evf[k] & 2:
            problems.append(f"event {ev.block(k)} of microbatch {ev.micro(k)} ends before it starts")
    for k in np.nonzero(evf & 12)[0].tolist():
        if evf[k] & 4:
            problems.append(f"unexpected block {ev.block(k)}")
        else:
            problems.append(f"unknown microbatch {ev.micro(k)}")
    sf = out["slot_flags"].cpu().numpy()[:n_slot]
    bad = np.nonzero(sf)[0]
    if bad.size:
        last = out["slot_last"].cpu().numpy()
        for x in bad.tolist():
            m, e = x // n_exp + 1, x % n_exp
            label, res = exp[e]
            if sf[x] & 1:
                problems.append(f"missing event: microbatch {m} block {label}")
                continue
            k = int(last[x])
            if sf[x] & 2:
                problems.append(f"block {label} of microbatch {m} on {ev.resource(k)}, expected {res}")
            if sf[x] & 4:
                d = _expected_duration(lc, N, merged, e, S)
                problems.append(f"block {label} of microbatch {m} runs {float(ev.end[k]) - float(ev.start[k]):.12g}, "
                                f"expected {d:.12g}")
    if problems:
        return problems

    # ---------------- phase 2 (scheduler.py:361-437)
    if 2 * M > _VAL_SORT_MAX:   # global-memory sort scratch for the overlap check
        cap = 1 << (2 * M - 1).bit_length()
        lanes = 2 * N - 1
        sk, se, si = f64(lanes * cap), f64(lanes * cap), i32(lanes * cap)
        a.sort_ks, a.sort_ke, a.sort_ki, a.sort_cap = sk.data_ptr(), se.data_ptr(), si.data_ptr(), cap
    _lib.check(lib.pp_validate_schedule(C.byref(a), 2, stream))
    stat = out["stat"].cpu().numpy()
    scal = out["scal"].cpu().numpy()
    if stat[0]:
        problems.append(f"first microbatch must enter stage 1 at time 0, starts at {float(scal[3]):.12g}")
    mn = out["mn_flags"].cpu().numpy()[:M * N].reshape(M, N)
    for m0, n0 in zip(*np.nonzero(mn)):
        m, n, f = int(m0) + 1, int(n0) + 1, int(mn[m0, n0])
        if n < N:
            if f & 1:
                problems.append(f"forward dependency violated at stage {n + 1}, microbatch {m}")
            if f & 2:
                problems.append(f"forward transfer on channel {n} starts before stage {n} output, microbatch {m}")
            if f & 4:
                problems.append(f"stage {n + 1} starts before channel {n} delivers, microbatch {m}")
            if f & 8:
                problems.append(f"backward dependency violated at stage {n}, microbatch {m}")
            if f & 16:
                problems.append(f"backward transfer on channel {n} starts before stage {n + 1} gradient, "
                                f"microbatch {m}")
            if f & 32:
                problems.append(f"stage {n} backward starts before channel {n} delivers, microbatch {m}")
        elif f & 64:
            problems.append(f"last-stage backward starts before its forward, microbatch {m}")
    arf = out["ar_flags"].cpu().numpy()[:N]
    for n in range(1, N + 1):
        f = int(arf[n - 1])
        if f & 1:
            problems.append(f"missing AllReduce for replicated stage {n}")
        if f & 2:
            problems.append(f"AllReduce of stage {n} starts before its last backward")
        if f & 4:
            problems.append(f"AllReduce of stage {n} has wrong duration")
        if f & 8:
            problems.append(f"AllReduce reported for unreplicated stage {n}")
    ovf = out["ov_flags"].cpu().numpy()
    if ovf.any():
        ovi = out["ov_idx"].cpu().numpy()
        names = [f"stage{r // 2 + 1}" if r % 2 == 0 else f"chan{r // 2 + 1}" for r in range(2 * N - 1)]
        for r in sorted(range(2 * N - 1), key=lambda r: names[r]):
            lo, hi = int(res_off[r]), int(res_off[r + 1])
            for j in np.nonzero(ovf[lo:hi])[0].tolist():
                p, q = int(ovi[lo + j - 1]), int(ovi[lo + j])
                problems.append(f"overlap on {names[r]}: ({ev.micro(p)},{ev.block(p)}) and "
                                f"({ev.micro(q)},{ev.block(q)})")
    if stat[1]:
        problems.append("barrier violated: backward-side work starts before all forward-side work done")
    if stat[2]:
        problems.append(f"makespan {float(schedule.makespan):.12g} does not match schedule contents "
                        f"{float(scal[0]):.12g}")
    return problems
