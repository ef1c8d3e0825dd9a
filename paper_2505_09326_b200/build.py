"""Build the in-tree FlashSign CUDA library for sm_100a.

    python -m paper_2505_09326_b200.build

Compiles ``csrc/flashsign_fwd.cu`` into ``_lib/libflashsign.so`` with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``).  The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OUT = os.path.join(OUT_DIR, "libflashsign.so")
SOURCES = ["flashsign_fwd.cu", "flashsign_prep.cu", "flashsign_gram.cu", "flashsign_exact.cu", "fs_host.cpp"]
DEPS = ["flashsign_fwd.cu", "flashsign_prep.cu", "flashsign_gram.cu", "flashsign_exact.cu", "fs_host.cpp", "sm100.cuh", os.path.join("..", "..", "include", "flashsign.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(os.path.join(CSRC, d)) <= t for d in DEPS)


TORCH_EXT = os.path.join(OUT_DIR, "fs_torch.so")
TORCH_EXT_SRC = os.path.join(CSRC, "fs_torch.cpp")


def build_torch_ext(force: bool = False, verbose: bool = False) -> str:
    """The PyTorch C++ extension (csrc/fs_torch.cpp -> _lib/fs_torch.so) over the C-ABI: compiled
    in-tree with torch's own flags, linked against libflashsign.so through an $ORIGIN rpath."""
    deps = [TORCH_EXT_SRC, os.path.join(HERE, "..", "include", "flashsign.h"), OUT]
    if not force and os.path.exists(TORCH_EXT) and all(os.path.getmtime(d) <= os.path.getmtime(TORCH_EXT)
                                                        for d in deps):
        return TORCH_EXT
    import sysconfig

    import torch
    from torch.utils import cpp_extension as ce

    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    inc = ce.include_paths(device_type="cuda") + [sysconfig.get_paths()["include"]]
    libdirs = ce.library_paths(device_type="cuda")
    tmp = TORCH_EXT + f".tmp{os.getpid()}"
    cmd = (["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
            "-DTORCH_EXTENSION_NAME=fs_torch", "-DTORCH_API_INCLUDE_EXTENSION_H", TORCH_EXT_SRC, "-o", tmp]
           + [f"-I{i}" for i in inc] + [f"-L{d}" for d in libdirs]
           + [f"-L{OUT_DIR}", "-lflashsign", "-Wl,-rpath,$ORIGIN", "-lc10", "-ltorch", "-ltorch_cpu", "-ltorch_python",
              "-lc10_cuda", "-ltorch_cuda", "-L/usr/local/cuda/lib64", "-lcudart"])
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, TORCH_EXT)
    return TORCH_EXT


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        build_torch_ext(force, verbose)
        return OUT
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = OUT + f".tmp{os.getpid()}"
    # FLASHSIGN_NVCC_EXTRA: diagnostic builds only (e.g. a longer mbarrier watchdog under racecheck)
    extra = os.environ.get("FLASHSIGN_NVCC_EXTRA", "").split()
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, OUT)
    build_torch_ext(True, verbose)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
