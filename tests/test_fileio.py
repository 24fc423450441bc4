"""File formats (reference fileio.py / test_fileio.py) on the host: JSON round
trips, parse errors, and the native trace writer (pp_format_trace) against
text the reference itself wrote (tests/golden/fileio.json)."""

import json
import math

import pytest

from helpers import fx, load, model_of

import paper_2204_10562_b200 as P
from paper_2204_10562_b200 import fileio as F
from paper_2204_10562_b200.model import LazyEvents


def _sim_cases():
    return {c["name"]: c for c in load("sim")["cases"] if "schedule" in c}


def _schedule_of(case):
    sc = case["schedule"]
    ev = tuple(P.ScheduleEvent(r, m, b, fx(s), fx(e)) for r, m, b, s, e in sc["events"])
    ar = tuple(P.AllReduceWindow(k, fx(s), fx(e)) for k, s, e in sc["allreduce"])
    return P.Schedule(events=ev, allreduce=ar, makespan=fx(sc["makespan"]))


def _plan_of(case):
    st = case["plan"]["stages"]
    return P.Plan(tuple(P.Stage(n + 1, a, b, tuple(d)) for n, (a, b, d) in enumerate(st)), case["plan"]["M"])


def test_format_number_matches_reference():
    for h, want in load("fileio")["format_number"]:
        assert F.format_number(fx(h)) == want
    assert F.format_number(3) == "3" and F.format_number(5.0) == "5" and F.format_number(1e9) == "1e+09"
    for bad in (math.inf, -math.inf, math.nan):
        with pytest.raises(P.ValidationError, match="non-finite"):
            F.format_number(bad)


def test_writers_match_reference_text():
    sims = _sim_cases()
    for c in load("fileio")["cases"]:
        case = sims[c["name"]]
        prof, clu, _ = model_of(case["input"])
        assert F.write_trace(None, _schedule_of(case)) == c["trace"], c["name"]
        assert F.save_profile(None, prof) == c["profile"]
        assert F.save_cluster(None, clu) == c["cluster"]
        assert F.save_plan(None, _plan_of(case)) == c["plan"]


def test_native_formatter_on_lazy_events_and_threads():
    """The LazyEvents path (arrays, no objects) and a multi-threaded split give
    the same bytes as Python's "%.9g"."""
    import numpy as np
    rng = np.random.default_rng(0)
    n = 50000
    res = [None, "stage1", "chan1", "stage2"]
    lab = [None, "fwd1", "comm_fwd1", "fwdbwd2"]
    pos = rng.integers(1, 4, n).astype(np.int32)
    m = rng.integers(1, 10 ** 6, n).astype(np.int32)
    s = np.exp(rng.uniform(-300, 300, n))
    e = s + rng.uniform(0, 1e3, n)
    sched = P.Schedule(events=LazyEvents(res, lab, m, pos, s, e),
                       allreduce=(P.AllReduceWindow(1, 0.25, 1 / 3),), makespan=float(e.max()))
    text = F.write_trace(None, sched)
    want = [f"# makespan {'%.9g' % sched.makespan}", F.TRACE_HEADER]
    want += [f"{res[q]},{a},{lab[q]},{'%.9g' % x},{'%.9g' % y}" for q, a, x, y in
             zip(pos.tolist(), m.tolist(), s.tolist(), e.tolist())]
    want.append("allreduce,0,allreduce_stage1,0.25,0.333333333")
    assert text == "\n".join(want) + "\n"


def test_trace_non_finite_is_rejected_in_output_order():
    ev = (P.ScheduleEvent("stage1", 1, "fwd1", 0.0, math.inf), P.ScheduleEvent("stage1", 2, "fwd1", math.nan, 1.0))
    with pytest.raises(P.ValidationError, match="non-finite number in output: inf"):
        F.write_trace(None, P.Schedule(events=ev, allreduce=(), makespan=1.0))
    with pytest.raises(P.ValidationError, match="non-finite number in output: -inf"):
        F.write_trace(None, P.Schedule(events=ev, allreduce=(), makespan=-math.inf))


def test_trace_round_trip_and_parse_errors(tmp_path):
    sims = _sim_cases()
    for name in ("tiny_split_pe_M2", "tiny_replicated", "rand0_pe"):
        sched = _schedule_of(sims[name])
        path = str(tmp_path / "t.csv")
        F.write_trace(path, sched)
        back = F.trace_to_schedule(F.read_trace(path))
        assert len(back.events) == len(sched.events) and back.allreduce == tuple(
            P.AllReduceWindow(w.stage, float("%.9g" % w.start), float("%.9g" % w.end)) for w in sched.allreduce)
    cases = [("resource,microbatch,block,start,end\nstage1,1,fwd1,0,1\n", "makespan"),
             ("# makespan eleven\nresource,microbatch,block,start,end\n", "bad makespan"),
             ("# makespan 11\nstage1,1,fwd1,0,1\n", "column header"),
             ("# makespan 11\nresource,microbatch,block,start,end\nstage1,1,fwd1\n", "malformed row"),
             ("# makespan 11\nresource,microbatch,block,start,end\nstage1,one,fwd1,0,1\n", "malformed row"),
             ("# makespan 0\nresource,microbatch,block,start,end\n", "no event rows")]
    for text, msg in cases:
        with pytest.raises(P.ValidationError, match=msg):
            F.parse_trace(text)
    with pytest.raises(P.ValidationError, match="cannot read"):
        F.read_trace(str(tmp_path / "absent.csv"))


def test_json_round_trips_and_errors(tmp_path):
    prof, clu, M = model_of(load("sim")["cases"][0]["input"])
    p = str(tmp_path / "p.json")
    F.save_profile(p, prof)
    assert F.load_profile(p) == prof
    data = json.loads(F.save_profile(None, prof))
    data["layers"].reverse()
    (tmp_path / "r.json").write_text(json.dumps(data))
    assert F.load_profile(str(tmp_path / "r.json")) == prof
    data["layers"][0]["fwd_s"] = -1.0
    (tmp_path / "n.json").write_text(json.dumps(data))
    with pytest.raises(P.ValidationError, match="negative"):
        F.load_profile(str(tmp_path / "n.json"))
    c = str(tmp_path / "c.json")
    F.save_cluster(c, clu)
    back = F.load_cluster(c)
    assert back == clu and back.bandwidth == clu.bandwidth
    plan = P.Plan((P.Stage(1, 1, 1, (1,)), P.Stage(2, 2, 2, (2,))), 2)
    F.save_plan(str(tmp_path / "plan.json"), plan)
    assert F.load_plan(str(tmp_path / "plan.json")) == plan
    (tmp_path / "res.json").write_text(json.dumps({"makespan": 11.0, "plan": json.loads(F.save_plan(None, plan))}))
    assert F.load_plan(str(tmp_path / "res.json")) == plan
    bad = [('{"name": "x"}', F.load_profile, "malformed profile"),
           ('{"gpus": [1, 2], "links": [{"a": 1}]}', F.load_cluster, "malformed cluster"),
           ("{nope", F.load_cluster, "not valid JSON"), ("[1, 2]", F.load_cluster, "top level"),
           ('{"microbatches": 2, "stages": [{"index": 1}]}', F.load_plan, "malformed plan")]
    for k, (text, fn, msg) in enumerate(bad):
        path = tmp_path / f"bad{k}.json"
        path.write_text(text)
        with pytest.raises(P.ValidationError, match=msg):
            fn(str(path))
