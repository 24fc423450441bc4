"""The reference's OWN test-suite, unchanged, against the drop-in.

``baseline/_ref/pipeplan_tests`` holds the reference's ``pkg/tests`` (staged by
``tools/stage_reference.py`` from /root/reference, git-ignored, shipped with the
repo snapshot).  It runs in a subprocess with ``dropin/`` first on
``PYTHONPATH``, so every ``import pipeplan`` in those files — and in their
conftest — resolves to ``dropin/pipeplan`` → ``paper_2204_10562_b200`` (CUDA).
The reference's brute-force ``oracle``, ``gantt`` and ``cli`` modules (out of
scope here) are executed from the staged reference copy as submodules of the
drop-in, so they too run on the drop-in's planner and types.

Every collected reference test must pass.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(REPO, "baseline", "_ref", "pipeplan_tests")
MODULES = ["test_partition.py", "test_scheduler.py", "test_planner.py", "test_cost.py", "test_ordering.py",
           "test_acceptance.py", "test_properties.py", "test_model.py", "test_baselines.py", "test_fileio.py",
           "test_oracle.py", "test_cli.py"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(SUITE):
        pytest.skip("reference suite not staged (python tools/stage_reference.py in the build container)")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "dropin"), REPO, os.path.join(REPO, "tests")] +
                                        ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


def test_suite_imports_the_dropin(tmp_path):
    probe = subprocess.run([sys.executable, "-c", "import pipeplan; print(pipeplan.IMPLEMENTATION)"],
                           cwd=tmp_path, env=_env(), capture_output=True, text=True)
    assert probe.stdout.strip() == "paper_2204_10562_b200", probe.stderr


@pytest.mark.parametrize("module", MODULES)
def test_reference_module_passes_on_dropin(module, tmp_path):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "refsuite_plugin",
                        "--durations=5",
                        os.path.join(SUITE, module)], cwd=tmp_path, env=_env(), capture_output=True, text=True,
                       timeout=1800)
    tail = "\n".join(r.stdout.splitlines()[-30:])
    assert r.returncode == 0, f"{module}:\n{tail}\n{r.stderr[-2000:]}"
    assert " passed" in tail and "failed" not in tail, tail
