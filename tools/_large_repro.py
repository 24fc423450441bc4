import sys, os, math, random
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import numpy as np
import test_gpu_parity as T
from helpers import model_of
import paper_2204_10562_b200 as P
from paper_2204_10562_b200 import _device, _lib
rng = random.Random(9)
specs = []
lu = lambda lo, hi: math.exp(rng.uniform(math.log(lo), math.log(hi)))
for L, V, M in ((150, 5, 4), (140, 9, 8), (3, 136, 2)):
    ids = rng.sample(range(1, 1000), V)
    specs.append(T._spec([lu(1e-3, 1.0) for _ in range(L)], [lu(1e-3, 2.0) for _ in range(L)],
                         [lu(1e6, 1e10) for _ in range(L)], [lu(1e5, 1e9) for _ in range(L - 1)],
                         [lu(1e5, 1e9) for _ in range(L - 1)], ids,
                         [(a, b, lu(1e8, 1e11)) for k, a in enumerate(ids) for b in ids[k + 1:]], M))
from paper_2204_10562_b200.partition import sum_flags
for sel in ([0], [1], [2], [0, 1], [0, 1, 2]):
    items = [(_device.pack(*model_of(specs[k])[:2]), specs[k]["M"], _lib.PP_ALLOW_REPLICATION | sum_flags(), None) for k in sel]
    db = _device.DeviceBatch(items, capture_events=True)
    db.run("spp")
    h = db.fetch()
    print(sel, "best_xi", h["best_xi"], "best_mk", h["best_mk"], "order", [list(h["order"][:5])], flush=True)
