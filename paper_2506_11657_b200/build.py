"""Build the sm_100a shared library in-tree (no JIT cache, no torch types).

    python -m paper_2506_11657_b200.build

produces paper_2506_11657_b200/libtem_b200.so from csrc/*.cu with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo``.
"""
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "tem_b200.cu"), os.path.join(HERE, "csrc", "tem_rkfit.cpp")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [os.path.join(ROOT, "include", "tem_b200.h")]
LIB = os.path.join(HERE, "libtem_b200.so")


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
           "-Xptxas", "-v" if verbose else "-O3", "-o", LIB + ".tmp"] + SRC
    extra = os.environ.get("TEM_NVCC_FLAGS", "").split()
    cmd = cmd[:-len(SRC) - 2] + extra + cmd[-len(SRC) - 2:]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
