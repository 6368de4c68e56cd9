"""Build helper: compiles csrc/*.cu into _lib/libharpia_b200.so for sm_100a.

Uses ``make`` in csrc/ (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo).
The .so is built in-tree so it travels with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent


def build_native(jobs: int = 8, verbose: bool = False) -> Path:
    nvcc = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    env = dict(os.environ, NVCC=nvcc)
    cmd = ["make", "-C", str(HERE / "csrc"), f"-j{jobs}"]
    if not verbose:
        cmd.append("-s")
    subprocess.run(cmd, check=True, env=env)
    return HERE / "_lib" / "libharpia_b200.so"


if __name__ == "__main__":
    print(build_native(verbose=True))
