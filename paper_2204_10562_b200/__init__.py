"""B200-native planning path of arXiv 2204.10562 ("pipeplan" drop-in).

Same public names and semantics as the reference package's planning path
(pipeplan/__init__.py:96-174): domain types, spp, PartitionSolver,
simulate_pe / simulate_with_order, RDO.  Planning arithmetic runs only in
libpipeplan_b200.so (sm_100a CUDA) — there is no CPU fallback; without a GPU
the planning calls raise _lib.BackendUnavailable.
"""

from .baselines import dataparallel_plan, gpipe_plan, gpipe_schedule, noreplication_plan
from .checker import validate_schedule
from .cost import (CostSummary, allreduce_time, block_duration, block_durations, channel_times, cost_summary, gamma,
                   interstage_comm_time, min_cross_bandwidth, min_pairwise_bandwidth)
from .fileio import (Trace, TraceRow, format_number, load_cluster, load_plan, load_profile, parse_trace, read_trace,
                     save_cluster, save_plan, save_profile, trace_to_schedule, write_trace)
from .model import (AllReduceWindow, Block, ClusterGraph, InterLayerEdge, LayerProfile, ModelProfile, Plan,
                    Schedule, ScheduleEvent, Stage, ValidationError, check_numeric_range, make_cluster,
                    plan_uses_all_gpus, validate_cluster, validate_plan, validate_profile)
from .ordering import DeviceOrdering, global_min_cut, rdo
from .partition import PartitionSolver, PrmResult, best_partition, prm
from .planner import BoundReport, SppResult, SweepEntry, bound_factor, phi, spp, spp_many, theorem1_report
from .scheduler import (ExecutionOrder, SchedulingError, build_block_list, compute_execution_order, lemma1_bound,
                        simulate_cycle_schedule, simulate_pe, simulate_pe_many, simulate_with_order)

from .warm import warmup

__version__ = "0.1.0"

__all__ = [
    "AllReduceWindow", "Block", "BoundReport", "ClusterGraph", "DeviceOrdering", "ExecutionOrder",
    "InterLayerEdge", "LayerProfile", "ModelProfile", "Plan", "PartitionSolver", "PrmResult", "Schedule",
    "ScheduleEvent", "SchedulingError", "SppResult", "Stage", "SweepEntry", "ValidationError",
    "best_partition", "bound_factor", "dataparallel_plan", "gpipe_plan", "gpipe_schedule",
    "noreplication_plan", "build_block_list", "check_numeric_range", "compute_execution_order",
    "global_min_cut", "lemma1_bound", "make_cluster", "phi", "plan_uses_all_gpus", "prm", "rdo",
    "simulate_pe", "simulate_pe_many", "simulate_with_order", "spp", "spp_many", "theorem1_report", "validate_cluster",
    "validate_plan", "validate_profile",
    "Trace", "TraceRow", "format_number", "load_cluster", "load_plan", "load_profile", "parse_trace", "read_trace",
    "save_cluster", "save_plan", "save_profile", "trace_to_schedule", "write_trace",
    "CostSummary", "allreduce_time", "block_duration", "block_durations", "channel_times", "cost_summary", "gamma",
    "interstage_comm_time", "min_cross_bandwidth", "min_pairwise_bandwidth", "simulate_cycle_schedule", "validate_schedule",
    "warmup",
]
