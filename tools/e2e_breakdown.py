"""Host-side breakdown of one spp_many() call on the C3 batch, or the C4 batch
with `c4` (run on the GPU box; `--profile` adds a cProfile of 5 calls)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2204_10562_b200 import planner, _device, workloads as W

specs = W.c4_batch(4096) if "c4" in sys.argv else W.c3_sweep()
models = W.models_of(specs)
planner.spp_many(models)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    items, packs = planner._items(models)
    t1 = time.perf_counter()
    db = _device.DeviceBatch(items, capture_events=True)
    t2 = time.perf_counter()
    db.run("spp")
    t3 = time.perf_counter()
    h = db.fetch()
    t4 = time.perf_counter()
    res = planner._decode_all(db, h, [it[1] for it in items], packs)
    t5 = time.perf_counter()
    print(f"validate+pack {1e3*(t1-t0):.1f} ms | DeviceBatch (H2D+alloc) {1e3*(t2-t1):.1f} | enqueue {1e3*(t3-t2):.1f} "
          f"| fetch (sync+D2H) {1e3*(t4-t3):.1f} | decode {1e3*(t5-t4):.1f} | total {1e3*(t5-t0):.1f}")

if "--profile" in sys.argv:
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        planner.spp_many(models)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
