"""Full-size C3 goldens (96 layers x 64 GPUs) from the LIVE Python reference.

Each case is one ``pipeplan.spp(profile, cluster, M)`` call at the headline
shape (reference ``planner.py:57-88`` → ``partition.py:113-142``).
One call takes hours of single-core CPU, so cases run as separate processes:

    python tests/golden/make_c3_full.py u8      # uniform, M = 8
    python tests/golden/make_c3_full.py j96_8   # jitter seed 96, M = 8

Output: ``tests/golden/c3_full_<case>.json`` in the same schema as
``spp.json`` (floats as ``float.hex``), plus the wall time of the reference
call and the interpreter / CPU it ran on.  Build container
only: it imports /root/reference, which the GPU box does not have.
"""

import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402  (puts the reference + repo on sys.path)
from paper_2204_10562_b200 import workloads as W  # noqa: E402

CASES = {
    "u8": dict(M=8, jitter_seed=None),
    "j96_8": dict(M=8, jitter_seed=96),
    "j96_256": dict(M=256, jitter_seed=96),
    "u32": dict(M=32, jitter_seed=None),
    "j96_64": dict(M=64, jitter_seed=96),
    "u128": dict(M=128, jitter_seed=None),
}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    name = sys.argv[1]
    spec = W.c3_gpt96(**CASES[name])
    t0 = time.time()
    case = G.spp_case(*G.ref_model(spec))
    case["case"] = name
    case["python"] = sys.version
    case["cpu"] = cpu_model()
    case["wall_seconds"] = time.time() - t0
    path = os.path.join(HERE, f"c3_full_{name}.json")
    with open(path, "w") as f:
        json.dump(case, f, separators=(",", ":"))
    print(f"{name}: spp {case['ref_seconds']:.1f} s -> {path}")


if __name__ == "__main__":
    main()
