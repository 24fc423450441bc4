import sys, time, cProfile, pstats
sys.path.insert(0, ".")
import torch
from paper_2204_10562_b200 import planner, _device, workloads as W
specs = W.c3_sweep(); models = W.models_of(specs)
planner.spp_many(models); torch.cuda.synchronize()
items, packs = planner._items(models)
def mk(): return _device.DeviceBatch(items, capture_events=True)
for _ in range(20): mk()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50): db = mk()
torch.cuda.synchronize()
print("DeviceBatch ms", (time.perf_counter() - t) / 50 * 1e3)
db.run("spp"); h = db.fetch()
t = time.perf_counter()
for _ in range(50): res = [planner._decode(db, h, k, items[k][1], packs[k]) for k in range(len(items))]
print("decode ms", (time.perf_counter() - t) / 50 * 1e3)
t = time.perf_counter()
for _ in range(50): h = db.fetch()
print("fetch (no device work) ms", (time.perf_counter() - t) / 50 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): db = mk()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(14)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): res = [planner._decode(db, h, k, items[k][1], packs[k]) for k in range(len(items))]
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(14)
