"""In-tree build of the sm_100a extension (nvcc, no JIT cache).

Produces ``paper_2412_16370_b200/libpospopcnt_b200.so`` from csrc/*.cu:
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared``
with the CUDA runtime linked statically, so the library does not depend on
whichever libcudart torch happens to have loaded.
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpospopcnt_b200.so")
# PP_CHECK_BOUNDS=1 build: every global load / bulk copy checked against the
# caller's range (pp_check_status); loaded through PP_LIB_PATH by the tests
CHECKED_LIB = os.path.join(HERE, "libpospopcnt_b200_checked.so")
SOURCES = ("pp_api.cu", "pp_count.cu", "pp_segmented.cu", "pp_categories.cu", "pp_gen.cu")
HEADERS = ("pp_device.cuh", "pp_internal.h")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
    "-Xptxas", "-v",
    "-cudart", "static",
    "-shared",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "pospopcnt_b200.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, lib=LIB, defines=()):
    if not force and not _stale(lib):
        return lib
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    tmp = lib + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, *srcs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(lib)}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


def build_checked(force=False, verbose=False):
    """The PP_CHECK_BOUNDS=1 variant (memory-safety evidence, tests only)."""
    return build(force, verbose, lib=CHECKED_LIB, defines=("PP_CHECK_BOUNDS=1",))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_checked(force="--force" in sys.argv))


def build_variant(out_path, defines):
    """Build an experimental variant (extra -D flags) to out_path (A/B timing)."""
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", out_path, *srcs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("variant build failed")
    return out_path
