"""Stage the reference package + its test-suite under baseline/_ref/ (git-ignored,
travels to the GPU box with the gpurun snapshot; never imported by the product).

    python tools/stage_reference.py [--force]

* baseline/_ref/pipeplan/        the reference installed with pip (offline,
                                 from a /tmp copy: /root/reference is read-only)
* baseline/_ref/pipeplan_tests/  the reference's pkg/tests, run UNCHANGED against
                                 the drop-in by tests/test_gpu_reference_suite.py

Needs /root/reference (build container only); a no-op when it is absent or
the staging already exists.
"""

import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DST = os.path.join(REPO, "baseline", "_ref")


def stage(force=False):
    if not os.path.isdir(REF):
        return False
    if force and os.path.isdir(DST):
        shutil.rmtree(DST)
    if not os.path.isfile(os.path.join(DST, "pipeplan", "planner.py")):
        with tempfile.TemporaryDirectory() as tmp:
            src = os.path.join(tmp, "pkg")
            shutil.copytree(REF, src)
            r = subprocess.run([sys.executable, "-m", "pip", "install", "-q", "--no-index", "--no-build-isolation",
                                "--find-links", "/opt/wheelhouse", "--target", DST, "--no-deps", src],
                               capture_output=True, text=True)
            if r.returncode != 0:
                print("reference install failed:", r.stderr[-400:])
                return False
    tdst = os.path.join(DST, "pipeplan_tests")
    os.makedirs(tdst, exist_ok=True)
    for f in sorted(os.listdir(os.path.join(REF, "tests"))):
        if f.endswith(".py"):
            shutil.copy2(os.path.join(REF, "tests", f), os.path.join(tdst, f))
    return True


if __name__ == "__main__":
    print("staged" if stage("--force" in sys.argv) else "reference not available")
