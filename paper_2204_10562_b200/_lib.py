"""ctypes binding of libpipeplan_b200.so (include/pipeplan_b200.h).

The planning path has no CPU fallback: importing the planning modules is
cheap, but the first planning call loads the library and requires a CUDA
device; if either is missing it raises :class:`BackendUnavailable` loudly.
"""

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PP_LIB_OVERRIDE") or os.path.join(HERE, "libpipeplan_b200.so")
CSRC = os.path.join(HERE, "csrc")
REPO = os.path.dirname(HERE)

NVCC_FLAGS = ["-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]

PP_ALLOW_REPLICATION = 1
PP_SUM_NAIVE = 2
PP_GIVEN_ORDER = 4
PP_SIM_FORWARD_BARRIER = 1
PP_SIM_PE_ORDER = 2
PP_SIM_CYCLE = 4
PP_SIM_COSTS_ONLY = 8
PP_LANE_COST_FIELDS = 7
PP_MAX_LAYERS = 4096
PP_MAX_GPUS = 512


class BackendUnavailable(RuntimeError):
    """The CUDA planning backend (libpipeplan_b200.so + a CUDA device) is missing."""


def build(verbose=False):
    """Compile the CUDA library in-tree for sm_100a."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-o", LIB_PATH, os.path.join(CSRC, "unity.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB_PATH


class PPInstance(C.Structure):
    _fields_ = [("L", C.c_int32), ("V", C.c_int32), ("M", C.c_int32), ("flags", C.c_int32),
                ("layer_off", C.c_int64), ("bw_off", C.c_int64), ("order_off", C.c_int64),
                ("sweep_off", C.c_int64), ("stage_off", C.c_int64), ("ws_off", C.c_int64),
                ("ev_off", C.c_int64), ("ar_off", C.c_int64)]


class PPBatch(C.Structure):
    _fields_ = [("n_inst", C.c_int32), ("max_L", C.c_int32), ("max_V", C.c_int32),
                ("inst", C.c_void_p),
                ("fwd", C.c_void_p), ("bwd", C.c_void_p), ("param", C.c_void_p),
                ("efwd", C.c_void_p), ("ebwd", C.c_void_p), ("bw", C.c_void_p),
                ("order", C.c_void_p),
                ("sweep_w", C.c_void_p), ("sweep_mk", C.c_void_p), ("sweep_bound", C.c_void_p),
                ("sweep_r", C.c_void_p),
                ("stage_ls", C.c_void_p), ("stage_le", C.c_void_p), ("stage_dlo", C.c_void_p),
                ("stage_dhi", C.c_void_p),
                ("best_xi", C.c_void_p), ("best_mk", C.c_void_p), ("phi", C.c_void_p),
                ("ev_start", C.c_void_p), ("ev_end", C.c_void_p),
                ("ar_start", C.c_void_p), ("ar_end", C.c_void_p),
                ("ws", C.c_void_p), ("gamma", C.c_void_p), ("ev_order", C.c_void_p),
                ("max_M", C.c_int32), ("ws_doubles", C.c_int64)]


class PPPlan(C.Structure):
    _fields_ = [("inst", C.c_int32), ("N", C.c_int32), ("M", C.c_int32), ("flags", C.c_int32),
                ("stage_off", C.c_int64), ("devoff_off", C.c_int64), ("queue_off", C.c_int64),
                ("lane_off", C.c_int64), ("ev_off", C.c_int64), ("ar_off", C.c_int64)]


class PPSimBatch(C.Structure):
    _fields_ = [("n_plan", C.c_int32), ("max_N", C.c_int32), ("plan", C.c_void_p),
                ("ls", C.c_void_p), ("le", C.c_void_p), ("dev_off", C.c_void_p), ("devs", C.c_void_p),
                ("q_off", C.c_void_p), ("q_items", C.c_void_p),
                ("makespan", C.c_void_p), ("bound", C.c_void_p), ("status", C.c_void_p),
                ("n_done", C.c_void_p), ("head", C.c_void_p),
                ("ev_start", C.c_void_p), ("ev_end", C.c_void_p),
                ("ar_start", C.c_void_p), ("ar_end", C.c_void_p), ("scratch", C.c_void_p),
                ("lane_cost", C.c_void_p), ("workload", C.c_void_p), ("cycles", C.c_void_p)]


EXPORTS = ("pp_version", "pp_last_error", "pp_device_count", "pp_layout", "pp_rdo", "pp_prm",
           "pp_pe_sweep", "pp_select", "pp_spp", "pp_prm_query", "pp_simulate", "pp_min_cut",
           "pp_launch_count", "pp_phi", "pp_peak_minmax", "pp_format_trace", "pp_validate_schedule",
           "pp_rdo_set_rounds", "pp_dp_set_persistent",
           "pp_dp_set_early_exit", "pp_step_trace", "pp_dp_set_combine",
           "pp_rdo_set_dedup")

_lib = None


def load(require_device=True):
    """Load the library (building it first only if the source tree is present
    and the .so is missing); with require_device, insist on a CUDA device."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BackendUnavailable(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a) first")
        lib = C.CDLL(LIB_PATH)
        _declare(lib)
        _lib = lib
    if require_device and _lib.pp_device_count() < 1:
        raise BackendUnavailable("no CUDA device visible: the planning path runs only on the GPU")
    return _lib


def _declare(L):
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.pp_version.restype = C.c_char_p
    L.pp_last_error.restype = C.c_char_p
    L.pp_device_count.restype = C.c_int
    L.pp_launch_count.restype = i64
    L.pp_layout.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.pp_layout.restype = C.c_int
    for name in ("pp_rdo", "pp_prm", "pp_pe_sweep", "pp_select", "pp_spp", "pp_phi"):
        fn = getattr(L, name)
        fn.argtypes = [vp, vp]
        fn.restype = C.c_int
    L.pp_prm_query.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp]
    L.pp_prm_query.restype = C.c_int
    L.pp_simulate.argtypes = [vp, vp, vp]
    L.pp_simulate.restype = C.c_int
    L.pp_min_cut.argtypes = [vp, i32, vp, i32, vp, vp, vp]
    L.pp_min_cut.restype = C.c_int
    L.pp_peak_minmax.argtypes = [vp, i32, vp, vp]
    L.pp_peak_minmax.restype = C.c_int
    L.pp_format_trace.argtypes = [C.c_int64, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, C.c_double, vp,
                                  C.c_int64, vp, i32]
    L.pp_format_trace.restype = C.c_int
    L.pp_validate_schedule.argtypes = [vp, i32, vp]
    L.pp_validate_schedule.restype = C.c_int
    L.pp_rdo_set_rounds.argtypes = [i32]
    L.pp_rdo_set_rounds.restype = C.c_int
    L.pp_dp_set_persistent.argtypes = [i32]
    L.pp_dp_set_persistent.restype = C.c_int
    L.pp_dp_set_early_exit.argtypes = [i32]
    L.pp_dp_set_early_exit.restype = C.c_int
    L.pp_rdo_set_dedup.argtypes = [i32]
    L.pp_rdo_set_dedup.restype = C.c_int
    L.pp_dp_set_combine.argtypes = [i32]
    L.pp_dp_set_combine.restype = C.c_int
    L.pp_step_trace.argtypes = [vp, i32]
    L.pp_step_trace.restype = C.c_int


def dp_persistent(mode) -> int:
    """DP schedule: 0 per-step launches, 3 one CTA per instance, 2 auto
    (default).  Returns the previous mode.  Results are identical either way."""
    prev = load(require_device=False).pp_dp_set_persistent(int(mode))
    if prev < 0:
        check(prev)
    return int(prev)


def dp_early_exit(on: bool) -> bool:
    """Toggle the combine's certified early exit; returns the previous setting."""
    prev = load().pp_dp_set_early_exit(1 if on else 0)
    if prev < 0:
        check(prev)
    return bool(prev)


def dp_combine(kind: int) -> int:
    """Per-step combine kernel: 1 crossing search, 0 exhaustive register
    tiles, 2 auto (default).  Returns the previous kind; results are identical."""
    return int(load(require_device=False).pp_dp_set_combine(int(kind)))


def rdo_dedup(mode: int) -> int:
    """RDO deduplication across a batch: 0 off, 1 auto (default), 2 always.
    Returns the previous mode; orders are identical either way."""
    return int(load(require_device=False).pp_rdo_set_dedup(int(mode)))


def rdo_rounds(rounds: int) -> int:
    """Set the speculative RDO round count (0 = sequential recursion only);
    returns the previous value.  The order is identical either way."""
    prev = load(require_device=False).pp_rdo_set_rounds(int(rounds))
    if prev < 0:
        check(prev)
    return prev


def check(rc):
    if rc != 0:
        msg = _lib.pp_last_error().decode() if _lib is not None else "library not loaded"
        raise RuntimeError(f"libpipeplan_b200 error {rc}: {msg}")


def launch_count():
    return int(load(require_device=False).pp_launch_count())
