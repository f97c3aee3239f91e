"""pytest plugin: run the reference's OWN test suite with the b200 kernel
registered in the reference's dispatch.

Loaded with ``-p refsuite_plugin`` by tests/test_gpu_ref_hw.py on the
reference tests staged under baseline/_ref/pkg_tests (scripts/
stage_reference.sh).  At configure time it imports the installed reference
(baseline/_ref, first on sys.path), appends ``B200Kernel`` to its registry
with ``paper_2412_16370_b200.ref_plugin.register`` -- no reference file is
edited -- so the reference's ``kernels`` fixture (pkg/tests/conftest.py:
28-30), ``get_kernel("b200")``, ``select_kernel``, the CLI and the bench
harness all see it.  With ``PP_REF_ONLY_B200=1`` every other kernel reports
unavailable, so kernel-parametrised tests (criterion 1's 491,776-call sweep)
run on b200 alone.
"""

import os


def pytest_configure(config):
    import pospopcnt as ref

    from paper_2412_16370_b200 import ref_plugin
    here = os.path.dirname(os.path.abspath(ref.__file__))
    want = os.environ.get("PP_REF_DIR")
    if want and not here.startswith(os.path.abspath(want)):
        raise RuntimeError(f"reference imported from {here}, expected under {want}")
    k = ref_plugin.register(ref)
    if not k.available():
        raise RuntimeError("b200 kernel registered but unavailable (no sm_100 device?)")
    if os.environ.get("PP_REF_ONLY_B200") == "1":
        for other in ref.kernels._registry():
            if other is not k:
                other.available = lambda: False  # instance override: hidden from fixtures
    config.pp_b200 = k


def pytest_report_header(config):
    return "refsuite_plugin: b200 kernel registered in the reference's dispatch"
