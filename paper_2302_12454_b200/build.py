"""In-tree build of libssqa_b200.so (CUDA engine + C ABI + C++ facade).

Everything is compiled for sm_100a only (``-gencode arch=compute_100a,
code=sm_100a``) with ``-lineinfo`` so ncu's source page maps to the code.
nvcc cross-compiles here without a GPU; the .so lands next to this file and
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libssqa_b200.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-Xptxas", "-v",
                     f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", f"-I{os.path.join(ROOT, 'include')}",
             f"-I{CSRC}", "-I/usr/local/cuda/include"]
# nlohmann/json (manifests in include/ssqa/bench.hpp), as the reference uses it;
# the image ships 3.11.3 with cuDNN's frontend headers
JSON_DIRS = [os.environ.get("SSQA_JSON_INCLUDE", ""),
             "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"]
JSON_INC = next((d for d in JSON_DIRS if d and os.path.exists(os.path.join(d, "nlohmann",
                                                                           "json.hpp"))), None)
if JSON_INC:
    CXX_FLAGS.append(f"-I{JSON_INC}")


def _sources():
    cu = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cpp"))
    if os.path.isdir(HOST):
        cpp += sorted(os.path.join(HOST, f) for f in os.listdir(HOST) if f.endswith(".cpp"))
    return cu, cpp


def _deps():
    out = []
    for d in (CSRC, HOST, os.path.join(ROOT, "include"), os.path.join(ROOT, "include", "ssqa")):
        if os.path.isdir(d):
            out += [os.path.join(d, f) for f in os.listdir(d)]
    return out


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.isfile(d))


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")


def build(force: bool = False, verbose: bool = False) -> str:
    cu, cpp = _sources()
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    log: list[str] = []
    objs = []
    for src in cu:
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        _run([NVCC, *CUDA_FLAGS, "-c", src, "-o", o], log)
        objs.append(o)
    for src in cpp:
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        _run(["g++", *CXX_FLAGS, "-c", src, "-o", o], log)
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda"], log)
    with open(os.path.join(ROOT, "build", "build.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
