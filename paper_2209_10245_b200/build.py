"""Builds libpoas_b200.so in-tree: C++20 planner/runtime (g++) + sm_100a
CUDA kernels (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo).

    python -m paper_2209_10245_b200.build [--force] [-j N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libpoas_b200.so"
CLI = PKG / "bin" / "poas"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC / 'include'}", f"-I{CSRC}", f"-I{CUDA_HOME / 'include'}"]
CXXFLAGS = ["-std=c++20", "-O3", "-g", "-fPIC", "-fopenmp", "-Wall", "-Wextra", "-Wno-unused-parameter"]
NVCCFLAGS = ["-std=c++20", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-fopenmp",
             "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def sources() -> list[Path]:
    out = []
    for sub in ("planner", "runtime", "kernels"):
        out += sorted((CSRC / sub).glob("*.cpp")) + sorted((CSRC / sub).glob("*.cu"))
    return out


def headers() -> list[Path]:
    hs = list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return hs


def obj_for(src: Path) -> Path:
    rel = src.relative_to(CSRC)
    return OBJ / (str(rel).replace("/", "__") + ".o")


def compile_one(src: Path) -> tuple[Path, str]:
    obj = obj_for(src)
    obj.parent.mkdir(parents=True, exist_ok=True)
    if src.suffix == ".cu":
        cmd = [NVCC, *NVCCFLAGS, *INCLUDES, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXXFLAGS, *INCLUDES, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> Path:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    srcs = sources()
    newest_hdr = max((h.stat().st_mtime for h in headers()), default=0.0)
    todo = []
    for s in srcs:
        o = obj_for(s)
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, newest_hdr):
            todo.append(s)
    logs = {}
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        for src, (obj, log) in zip(todo, ex.map(compile_one, todo)):
            logs[src] = log
    if verbose:
        for src, log in logs.items():
            if log.strip():
                print(f"== {src.name}\n{log}", file=sys.stderr)
    objs = [obj_for(s) for s in srcs]
    if todo or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs),
               "-Xcompiler", "-fopenmp", "-lgomp", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    # The `poas` CLI: its own main, linked against the same objects.
    cli_src = CSRC / "tools" / "poas_cli.cpp"
    cli_obj = obj_for(cli_src)
    if force or not cli_obj.exists() or cli_obj.stat().st_mtime < max(cli_src.stat().st_mtime, newest_hdr):
        compile_one(cli_src)
    if not CLI.exists() or CLI.stat().st_mtime < max(o.stat().st_mtime for o in [*objs, cli_obj]):
        CLI.parent.mkdir(exist_ok=True)
        tmp = CLI.with_suffix(".tmp")
        cmd = [NVCC, *ARCH, "-o", str(tmp), str(cli_obj), *map(str, objs),
               "-Xcompiler", "-fopenmp", "-lgomp", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, CLI)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j, verbose=a.v))


if __name__ == "__main__":
    main()
