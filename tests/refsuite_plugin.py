"""pytest plugin for the reference-suite runner (tests/test_gpu_reference_suite.py):
warm the drop-in up once per process (CUDA context, library, kernels) before
the first reference test, as a long-lived planning process would be — the
reference's per-test deadlines (hypothesis 200 ms, test_acceptance.py:82 1 s)
assume a warm interpreter, not CUDA start-up."""


def pytest_sessionstart(session):
    import pipeplan
    pipeplan.warmup()
