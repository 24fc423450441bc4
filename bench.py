#!/usr/bin/env python
"""Planning throughput benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (config.workload = "c3_gpt96_8x8_msweep"): the C3 planning batch of
BASELINE.json configs[2] — a GPT-style 96-layer profile on a 64-GPU two-tier
topology (8 nodes x 8, 450 GB/s NVLink inside a node, 12.5 GB/s = 100 Gb
between nodes), planned for every microbatch count M in 8..256, once with the
uniform profile and once with a jittered one: 12 spp() instances per GPU per
step.  A step = one full spp() over the batch (RDO, DP tables, wavefront DP,
backtrack of every xi, batched PE simulation of every feasible plan,
selection, replay of the chosen plans with event capture).

value  = instances / s over all ranks, device time (CUDA events on the
         library's stream), inputs resident in HBM, L2 flushed between steps.
e2e    = the same through the public drop-in API spp_many() with host
         profile/cluster objects: packing, one pinned H2D copy, kernels, D2H
         of every result, and the Python SppResult objects (schedule events
         included), timed on the host clock.
p50_latency_ms = single-instance spp() latency (C3, M = 32) on the device.

Multi-GPU: ``--gpus N`` launches N ranks itself (re-exec under
torch.distributed.run when WORLD_SIZE is unset; the driver's own torchrun
launch is used as is), one process per GPU, NCCL with INIT logging on stderr.
* c3 (headline, weak scaling): each rank plans its own 12-instance batch
  (jitter seed 96 + rank).
* c4 (strong scaling): the fixed 4096-instance batch split round-robin.
* c5 (strong scaling): the 256 candidate plans (xi = 1..256) striped across
  ranks (xi = rank + 1, rank + 1 + N, ...).
Instances and candidates are independent, so there is no data-path
collective; the one real exchange is the global arg-min of the chosen plans:
an NCCL all_gather of the per-rank counts, then of the padded
(makespan, xi, instance) records (distributed.global_best), reported as
"global_best".

--impl reference times the reference CPU planner restated in C (oracle/, the
reference itself is Python and cannot travel to the GPU box) on the host
cores: each timed step plans one C3 instance per worker thread.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = "c3_gpt96_8x8_msweep"
METRIC = "planning instances/sec and p50 plan latency (96-layer, 64-GPU topo) at 1-8 B200"
UNIT = "instances/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--profile-steps", type=int, default=0, help="(for ncu) run N untimed steps and exit")
    ap.add_argument("--workload", default="c3", choices=["c3", "c4", "c5"],
                    help="c3 = the headline (BASELINE.json metric); c4/c5 = secondary configs (strong scaling)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="TEST ONLY: every rank on cuda:0 with gloo collectives (exercises the N-rank "
                         "launch / sharding / min-loc path on a one-GPU box; not a scaling number)")
    ap.add_argument("--clock-soak-s", type=float, default=1.0,
                    help="untimed load steps right before the timed region, sampled for clocks with it")
    return ap.parse_args()


def maybe_self_launch(args):
    """--gpus N > 1 outside torchrun: re-exec this script under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous)."""
    if "WORLD_SIZE" in os.environ:
        ws = int(os.environ["WORLD_SIZE"])
        if args.impl == "ours" and ws != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
            sys.exit(2)
        return
    if args.gpus <= 1 or args.impl == "reference":
        return
    import socket
    import torch
    if torch.cuda.device_count() < args.gpus and not args.share_gpu:
        print(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} visible", file=sys.stderr)
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


SHARE_GPU = "--share-gpu" in sys.argv


def init_dist(local):
    """NCCL process group (one rank per GPU); INIT logs to stderr so the
    communicator's rank count is visible.  --share-gpu: gloo (test only)."""
    import torch
    import torch.distributed as dist
    if SHARE_GPU:
        dist.init_process_group("gloo")
        return
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def batch_specs(rank):
    from paper_2204_10562_b200 import workloads as W
    return W.c3_sweep(jitter_seeds=(None, 96 + rank))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def soak(step, seconds):
    """Untimed load for `seconds` (clock sampling under load before the timed region)."""
    import torch
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds or n < 3:
        step()
        n += 1
        if n % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": len(os.sched_getaffinity(0)), "python": sys.version.split()[0],
            "sum_mode": "neumaier" if sys.version_info >= (3, 12) else "naive"}


# ----------------------------------------------------------------------------- our arm
def t_fact(L, V):
    """Factored candidate count of one DP: sum over xi of
    A*K(K+1)(K+2)/6 + A(A+1)/2 * K(K+1)/2, A = L-xi+1, K = V-xi+1."""
    tot = 0
    for xi in range(2, min(L, V) + 1):
        A, K = L - xi + 1, V - xi + 1
        tot += A * K * (K + 1) * (K + 2) // 6 + A * (A + 1) // 2 * K * (K + 1) // 2
    return tot


def sim_executions(res_sweep, M):
    return sum(M * (4 * e.stage_count - 3) for e in res_sweep if e.feasible)


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        init_dist(local)
    from paper_2204_10562_b200 import _device, _lib, spp_many
    from paper_2204_10562_b200.distributed import global_best
    from paper_2204_10562_b200 import workloads as W
    from paper_2204_10562_b200.partition import sum_flags

    dev = torch.device("cuda", local)
    specs = batch_specs(rank)
    models = W.models_of(specs)   # one cluster object, two profile objects (as a user would)
    items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in models]
    db = _device.DeviceBatch(items, capture_events=True)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()

    if args.profile_steps:
        for _ in range(args.profile_steps):
            db.run("spp")
        torch.cuda.synchronize()
        return

    for _ in range(max(args.warmup, 3)):
        db.run("spp")
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, per-step CUDA events, L2 flushed between steps
    clocks = ClockSampler(local)
    clocks.start()
    soak(lambda: (flush.zero_(), db.run("spp")), args.clock_soak_s)
    n0 = _lib.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        db.run("spp")
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - n0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    dev_ms = sum(step_ms)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    n_inst = len(specs) * world
    value = n_inst * args.steps / (max_ms / 1e3)

    # ---- global best plan: NCCL min-loc over (makespan, xi, instance)
    h = db.fetch()
    import numpy as np
    gb = global_best(h["best_mk"], h["best_xi"], np.arange(len(specs)) + rank * len(specs))
    gbest = {"makespan": gb[0], "xi": gb[1], "instance": gb[2]}

    # ---- phase split (one more step, events between C-ABI calls on the same stream)
    phase = phase_split(db, flush, stream)

    # ---- roofline of the dominant phase (the DP): fp64 min/max pipe
    best_peak = live_minmax_peak(dev, stream)
    dp_ops = 2 * sum(t_fact(s.L, s.V) for s in specs)   # one max + one min per factored candidate
    dp_achieved = dp_ops / (phase["dp"] / 1e3)
    traffic, traffic_src = None, None
    for name in ("r02b_dp_traffic_warm.json", "r02_dp_traffic_warm.json", "ncu_dp_traffic.json"):   # newest first
        tpath = os.path.join(REPO, "profiles", name)
        if os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                traffic, traffic_src = tj.get("dram_bytes_per_step"), f"profiles/{name}: {tj.get('what', '')}"
                break
            except (OSError, ValueError):
                pass
    roofline = {"bound": "fp64_minmax", "kernel": "pp_prm (k_combine + k_expand wavefront)",
                "achieved": dp_achieved / 1e12, "peak": best_peak / 1e12, "unit": "Tminmax/s",
                "frac": dp_achieved / best_peak, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "k_peak_minmax measured live (no fp64 min/max figure in MEASURED_PEAKS.json)",
                "algorithmic_ops_per_step": dp_ops,
                "phase_ms": phase}

    # ---- single-instance p50 latency (C3, M = 32), device-resident
    one = _device.DeviceBatch([items[2]], capture_events=True)
    for _ in range(3):
        one.run("spp")
    lat = []
    for _ in range(max(5, min(args.steps, 20))):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream); one.run("spp"); b.record(stream)
        torch.cuda.synchronize()
        lat.append(a.elapsed_time(b))
    p50 = statistics.median(lat)

    # ---- e2e through the public API (host objects in, SppResult objects out)
    spp_many(models)
    torch.cuda.synchronize()
    e2e_t = []
    h2d = db.h2d_bytes()
    d2h = db.d2h_bytes()
    for _ in range(max(10, min(args.steps, 30))):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = spp_many(models)
        t1 = time.perf_counter()
        e2e_t.append(t1 - t0)
    tt = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_value = n_inst * len(e2e_t) / float(tt.item())
    e2e_lat = []
    for _ in range(5):
        t0 = time.perf_counter()
        spp_many([models[2]])
        e2e_lat.append(time.perf_counter() - t0)
    sim_exec = sum(sim_executions(r.sweep, r.plan.microbatch_count) for r in res)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(specs, args.cpu_threads)
        cpu["python_reference"] = python_reference_timing()
        cpu["host"] = host_info()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "instances_per_gpu": len(specs), "layers": 96, "gpus_in_topology": 64,
                   "topology": "8x8 two-tier (450e9 / 12.5e9 B/s)", "microbatches": [8, 16, 32, 64, 128, 256],
                   "profiles": ["uniform", f"jitter(seed 96+rank)"], "parallelism": f"instances sharded x{world}",
                   "l2": "flushed (256 MB write) between timed steps"},
        "p50_latency_ms": p50,
        "p50_latency_config": "one C3 instance (M=32), device-resident",
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "calls": len(e2e_t), "median_call_ms": 1e3 * statistics.median(e2e_t),
                "p50_latency_ms": 1e3 * statistics.median(e2e_lat), "api": "paper_2204_10562_b200.spp_many"},
        "gpu_launches": launches,
        "roofline": roofline,
        "sim_block_executions_per_step": sim_exec,
        "global_best": gbest,
        "clocks": clk,
        "cpu_baseline": cpu,
        "host": host_info(),
    }
    if SHARE_GPU:
        line["share_gpu_test"] = "all ranks on cuda:0, gloo collectives: exercises the N-rank path, not a scaling number"
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- CPU legs
def _oracle_instances(specs):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import numpy as np
    import oracle as O
    out = []
    for s in specs:
        ids = sorted(s.gpu_ids)
        pos = {g: k for k, g in enumerate(ids)}
        bw = np.zeros((len(ids), len(ids)))
        for a, b, w in s.links:
            bw[pos[a], pos[b]] = bw[pos[b], pos[a]] = w
        out.append(O.Instance(s.fwd, s.bwd, s.param, s.efwd, s.ebwd, bw, s.M))
    return O, out


def host_threads(req=0):
    """All host threads, capped at 64 (each C3 oracle DP holds a 0.33 GB dense table)."""
    n = len(os.sched_getaffinity(0))
    return max(1, min(req or n, n, 64))


def cpu_baseline(specs, threads=0):
    """The oracle (C port of the reference planner) on a bounded sample: one
    C3 instance per worker thread, all host threads."""
    O, insts = _oracle_instances(specs)
    nt = host_threads(threads)
    sample = [insts[k % len(insts)] for k in range(nt)]
    t0 = time.perf_counter()
    O.spp_batch(sample, nt)
    dt = time.perf_counter() - t0
    return {"value": len(sample) / dt, "unit": UNIT, "cores": nt, "kind": "port",
            "sample": f"{len(sample)} C3 instances (96 layers x 64 GPUs, M cycling 8..256), one per thread, "
                      f"{dt:.1f} s", "python_reference_note": "pure-Python reference ~2.2 h per C3 instance "
                      "(SURVEY.md §6 extrapolation), not runnable on the GPU box"}


def python_reference_timing():
    """The untouched Python reference (pipeplan.spp from baseline/_ref, staged by
    tools/stage_reference.py), timed in-process on one core for C1 and C2
    (single-threaded like the reference).  None when the staged
    copy is absent.  Measured in a subprocess so its `pipeplan` never meets ours."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "pipeplan", "planner.py")):
        return None
    code = r"""
import json, statistics, sys, time
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[2])
import pipeplan as P
from paper_2204_10562_b200 import workloads as W
out = {"python": sys.version.split()[0], "module": P.__file__}
for name, spec, reps in (("C1", W.c1_vgg19(), 7), ("C2", W.c2_bert24(), 3)):
    layers = tuple(P.LayerProfile(k + 1, f, b, p) for k, (f, b, p) in enumerate(zip(spec.fwd, spec.bwd, spec.param)))
    edges = tuple(P.InterLayerEdge(k + 1, k + 2, a, b) for k, (a, b) in enumerate(zip(spec.efwd, spec.ebwd)))
    prof = P.ModelProfile(spec.name, 1, layers, edges)
    clu = P.make_cluster(spec.gpu_ids, spec.links)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); P.spp(prof, clu, spec.M); ts.append(time.perf_counter() - t0)
    out[name] = {"p50_s": statistics.median(ts), "reps": reps}
print(json.dumps(out))
"""
    try:
        r = subprocess.run([sys.executable, "-c", code, ref, REPO], capture_output=True, text=True, timeout=300)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError):
        return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    specs = batch_specs(0)
    O, insts = _oracle_instances(specs)
    from paper_2204_10562_b200 import workloads as W
    _, warm = _oracle_instances([W.c2_bert24()])
    nt = host_threads(args.cpu_threads)
    for _ in range(args.warmup):
        O.spp_batch(warm, 1)
    times = []
    k = 0
    for _ in range(args.steps):
        sample = [insts[(k + j) % len(insts)] for j in range(nt)]
        k += nt
        t0 = time.perf_counter()
        O.spp_batch(sample, nt)
        times.append(time.perf_counter() - t0)
    value = nt * args.steps / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "layers": 96, "gpus_in_topology": 64,
                   "step": f"{nt} C3 instances, one per host thread"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nt, "kind": "port",
                         "sample": f"{nt} C3 instances per step x {args.steps} steps",
                         "python_reference": python_reference_timing(), "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_secondary(args):
    """Secondary configs, strong scaling over --gpus N (fixed total work):
    c4 — 4096 random 32-layer profiles x random 16-GPU cliques, M = 32,
         split round-robin across ranks: spp instances/s;
    c5 — the 256 candidate plans (xi = 1..256, even split on the RDO order) of a
         1024-layer chain on a 256-GPU clique, M = 512, striped across ranks:
         simulated block executions/s.  `value` times the simulation kernel alone
         (plans uploaded once, outside the timed region; RDO excluded as in
         SURVEY.md §8d); `e2e` times the public path per step (plan packing +
         H2D, the kernel, D2H of every makespan)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2204_10562_b200 import _device, _lib, rdo, spp_many
    from paper_2204_10562_b200 import workloads as W
    from paper_2204_10562_b200.distributed import global_best, shard
    from paper_2204_10562_b200.partition import sum_flags
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        init_dist(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def timed(fn):
        for _ in range(max(args.warmup, 3)):
            fn()
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        soak(lambda: (flush.zero_(), fn()), args.clock_soak_s)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n0 = _lib.launch_count()
        evs = []
        for _ in range(args.steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream); fn(); b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        launches = _lib.launch_count() - n0
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
        tot = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        return float(tot.item()), launches, clk

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak = live_minmax_peak(dev, stream)
    O, _ = _oracle_instances([]) if rank == 0 else (None, None)
    if args.workload == "c4":
        n_total = 4096
        mine = shard(n_total, rank, world)
        specs = [W.c4_instance(k) for k in mine]
        models = [s.to_model() for s in specs]
        items = [(_device.pack(p, c), M, _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for p, c, M in models]
        db = _device.DeviceBatch(items, capture_events=True)
        max_ms, launches, clk = timed(lambda: db.run("spp"))
        value = n_total * args.steps / (max_ms / 1e3)
        h = db.fetch()
        gb = global_best(h["best_mk"], h["best_xi"], np.array(mine))
        # phase split (this rank): DP share of the step
        phase = phase_split(db, flush, stream)
        dp_ops = 2 * len(specs) * t_fact(32, 16)
        dp_rate = dp_ops / (phase["dp"] / 1e3)
        # e2e: host objects -> SppResult objects through the public API
        spp_many(models)
        torch.cuda.synchronize()
        e2e = []
        for _ in range(max(3, min(args.steps, 5))):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            spp_many(models)
            e2e.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(e2e))
        line = {"metric": "C4 batched planning throughput", "value": value, "unit": "instances/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c4_4096x(L32,V16,M32)", "instances_total": n_total,
                           "parallelism": f"instances round-robin over {world} ranks",
                           "l2": "flushed (256 MB write) between timed steps"},
                "gpu_launches": launches,
                "e2e": {"value": n_total * len(e2e) / e2e_s, "unit": "instances/s",
                        "h2d_bytes_per_step": db.h2d_bytes(), "d2h_bytes_per_step": db.d2h_bytes(),
                        "api": "paper_2204_10562_b200.spp_many"},
                "roofline": {"bound": "fp64_minmax", "kernel": "k_dp_inst2 (instance-per-CTA DP, operands in shared memory)",
                             "achieved": dp_rate / 1e12, "peak": peak / 1e12, "unit": "Tminmax/s",
                             "frac": dp_rate / peak, "traffic": None, "algorithmic_ops_per_step": dp_ops,
                             "phase_ms": phase, "peak_source": "k_peak_minmax measured live"},
                "global_best": {"makespan": gb[0], "xi": gb[1], "instance": gb[2]},
                "clocks": clk, "host": host_info()}
        if rank == 0 and not args.no_cpu_baseline:
            _, sample = _oracle_instances(W.c4_batch(64))
            nt = host_threads(args.cpu_threads)
            t0 = time.perf_counter(); O.spp_batch(sample, nt); dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": len(sample) / dt, "unit": "instances/s", "cores": nt, "kind": "port",
                                    "sample": f"64 C4 instances on {nt} threads, {dt:.1f} s"}
    else:
        spec = W.c5_instance()
        profile, cluster, M = spec.to_model()
        order = rdo(cluster).order
        ids = sorted(spec.gpu_ids)
        pos = {g: k for k, g in enumerate(ids)}
        packed = _device.pack(profile, cluster)
        db = _device.DeviceBatch([(packed, M, sum_flags(), None)], capture_events=False, workspace=False)
        xis = [k + 1 for k in shard(256, rank, world)]

        def plans():
            return [_device.SimPlan(inst=0, M=M, stages=[(a, b, [pos[g] for g in d]) for a, b, d in
                                                         W.even_split_plan(spec.L, order, xi)],
                                    flags=_lib.PP_SIM_PE_ORDER) for xi in xis]
        sr = _device.SimRun(db, plans(), capture_events=False, launch=False)
        max_ms, launches, clk = timed(sr.launch)
        execs = sum(M * (4 * xi - 3) for xi in range(1, 257))
        value = execs * args.steps / (max_ms / 1e3)
        recs = sr.fetch()
        gb = global_best([r["makespan"] for r in recs], xis, [0] * len(xis))
        # e2e: host plan packing + upload + kernel + D2H of the makespans, host clock
        e2e = []
        for _ in range(max(3, min(args.steps, 10))):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            r2 = _device.SimRun(db, plans(), capture_events=False)
            r2.d_f[:len(xis)].cpu()
            e2e.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(e2e))
        chain = M + 4 * max(xis) - 4
        line = {"metric": "C5 candidate-plan simulation throughput", "value": value, "unit": "block executions/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c5_256plans_1024layers_256gpus_M512", "block_executions_per_step": execs,
                           "parallelism": f"candidates xi striped over {world} ranks",
                           "timed": "k_sim_plans alone, plans resident (uploaded once)", "rdo": "excluded"},
                "gpu_launches": launches,
                "e2e": {"value": execs * len(e2e) / e2e_s, "unit": "block executions/s",
                        "h2d_bytes_per_step": int(sr._keep.numel() * 4), "d2h_bytes_per_step": 8 * len(xis),
                        "api": "_device.SimRun (plan packing + upload + kernel + makespans D2H)"},
                "roofline": {"bound": "latency", "kernel": "k_sim_plans (PE pass sweep)",
                             "critical_chain_passes": chain,
                             "ns_per_chain_pass": 1e6 * (max_ms / args.steps) / chain,
                             "note": "one plan per CTA; the xi = 256 plan's M + 4N - 4 dependent passes "
                                     "bound the kernel"},
                "global_best": {"makespan": gb[0], "xi": gb[1]},
                "clocks": clk, "host": host_info()}
        if rank == 0 and not args.no_cpu_baseline:
            _, (oi,) = _oracle_instances([spec])
            nt = host_threads(args.cpu_threads)
            oplans = [O.Plan([(a, b, tuple(pos[g] for g in d)) for a, b, d in W.even_split_plan(spec.L, order, xi)],
                             M) for xi in range(1, 257, 8)]
            t0 = time.perf_counter(); O.simulate_pe_batch(oi, oplans, nt); dt = time.perf_counter() - t0
            cexec = sum(M * (4 * xi - 3) for xi in range(1, 257, 8))
            line["cpu_baseline"] = {"value": cexec / dt, "unit": "block executions/s", "cores": nt, "kind": "port",
                                    "sample": f"32 of the 256 plans (every 8th xi) on {nt} threads, {dt:.1f} s"}
    if rank == 0:
        if SHARE_GPU:
            line["share_gpu_test"] = "all ranks on cuda:0, gloo collectives: exercises the N-rank path, not a scaling number"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def live_minmax_peak(dev, stream):
    """fp64 compare-select peak (k_peak_minmax: 8 independent min/max chains per thread)."""
    import ctypes as C
    import torch
    from paper_2204_10562_b200 import _lib
    lib = _lib.load()
    out = torch.empty(1, dtype=torch.float64, device=dev)
    nops = C.c_int64()
    best = 0.0
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _lib.check(lib.pp_peak_minmax(C.c_void_p(out.data_ptr()), 4096, C.byref(nops), C.c_void_p(stream.cuda_stream)))
        b.record(stream)
        torch.cuda.synchronize()
        best = max(best, nops.value / (a.elapsed_time(b) / 1e3))
    return best


def phase_split(db, flush, stream):
    """Device time per spp phase (min of 3), events between the C-ABI calls."""
    import torch
    phase = {}
    for _ in range(3):
        flush.zero_()
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        marks[0].record(stream); db.run("phi"); db.run("rdo")
        marks[1].record(stream); db.run("prm")
        marks[2].record(stream); db.run("sweep")
        marks[3].record(stream); db.run("select")
        marks[4].record(stream)
        torch.cuda.synchronize()
        for k, nm in enumerate(("rdo", "dp", "simulate", "select")):
            phase.setdefault(nm, []).append(marks[k].elapsed_time(marks[k + 1]))
    return {k: min(v) for k, v in phase.items()}


def main():
    args = parse()
    maybe_self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload != "c3":
        run_secondary(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
