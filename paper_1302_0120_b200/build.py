"""Build libphasemask_b200.so in-tree for sm_100a.

    python -m paper_1302_0120_b200.build [--force] [--jobs N]

Compiles csrc/pm_inst.cu once per (precision, log2 length) plus the table
and C-ABI translation units, in parallel, with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (no fast-math:
the fp64 path needs IEEE sqrt/div, the fp32 path matches numpy's rounding),
and links them into ``paper_1302_0120_b200/lib/libphasemask_b200.so`` with
the CUDA runtime linked statically. Objects are cached under
``paper_1302_0120_b200/build/`` and rebuilt when a source or header changes.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libphasemask_b200.so"
INCLUDE = PKG.parent / "include"
MAX_LG = 12

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         f"-I{CSRC}", f"-I{INCLUDE}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build phasemask_b200")


# log2 points per thread of the row / column kernels and the persistent
# kernel's CTA size, per precision and size (DESIGN.md "Kernel
# configuration"); override every size at once for experiments with
# PM_LGR="f32row,f32col,f64row,f64col" and PM_SOLVE_NT="f32,f64".
# Measured on B200 (profiles/): radix-4 / radix-8 with 256-thread CTAs
# for 256^2 / 512^2 (latency-bound: short chains),
# radix-32 rows and columns with a 256-thread persistent CTA at 1024^2 fp32,
# radix-16 and 512 threads for the HBM-resident 2048^2 / 4096^2 grids and
# for fp64.
def default_config(tag: str, lg: int) -> tuple[int, int, int]:
    """(log2 points per thread of rows, of columns, persistent CTA size)."""
    if lg <= 8:
        return (2, 2, 256)          # short dependency chains (256^2: 6.4 / 8.5 us per iteration f32 / f64,
                                    # vs 8.4 / 9.9 with 128-thread CTAs; scripts/variants_small.sh)
    if lg == 9:
        return (3, 3, 256)
    if tag == "f32":
        return (5, 5, 256) if lg == 10 else (4, 4, 512)
    return (4, 3, 512)


def _config(tag: str, lg: int) -> tuple[int, int, int]:
    row, col, nt = default_config(tag, lg)
    only = os.environ.get("PM_XONLY")                  # experiment overrides for these units only
    if only and f"{tag}_{lg}" not in only.split(","):
        return row, col, nt
    env = os.environ.get("PM_LGR")
    if env:
        a = [int(x) for x in env.split(",")]
        row, col = (a[0], a[1]) if tag == "f32" else (a[2], a[3])
    env = os.environ.get("PM_SOLVE_NT")
    if env:
        a = [int(x) for x in env.split(",")]
        nt = a[0] if tag == "f32" else a[-1]
    return row, col, nt


def _units(build_dir):
    units = []
    for f64 in (0, 1):
        tag = "f64" if f64 else "f32"
        for lg in range(MAX_LG + 1):
            row, col, nt = _config(tag, lg)
            roll = int(os.environ.get("PM_ROLL", "0"))
            pf = int(os.environ.get("PM_PF", "0"))
            xd = os.environ.get("PM_XDEFS", "").split()        # experiment macros (-DNAME=V ...)
            only = os.environ.get("PM_XONLY")                  # e.g. "f32_10,f64_8": macros for these units only
            if only and f"{tag}_{lg}" not in only.split(","):
                xd = []
            xs = "".join("_" + d.lstrip("-D").replace("=", "") for d in xd)
            units.append((CSRC / "pm_inst.cu", build_dir / f"pm_inst_{tag}_{lg}_{row}{col}_{nt}_r{roll}_p{pf}{xs}.o",
                          [f"-DPM_F64={f64}", f"-DPM_LG={lg}", f"-DPM_LGR_ROW={row}", f"-DPM_LGR_COL={col}",
                           f"-DPM_SOLVE_NT={nt}", f"-DPM_ROLL={roll}", f"-DPM_PF={pf}", *xd]))
    units.append((CSRC / "pm_table.cu", build_dir / "pm_table.o", []))
    units.append((CSRC / "pm_capi.cu", build_dir / "pm_capi.o", []))
    return units


def _deps_mtime() -> float:
    files = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    files += list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return max(f.stat().st_mtime for f in files)


def _compile(unit, force: bool, verbose: bool):
    src, obj, defs = unit
    if not force and obj.exists() and obj.stat().st_mtime >= _deps_mtime():
        return obj, None
    cmd = [nvcc(), *ARCH, *FLAGS, *defs, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {obj.name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr if verbose else None


def build(force: bool = False, jobs: int | None = None, verbose: bool = False,
          out: Path | None = None) -> Path:
    lib = Path(out) if out else LIB
    BUILD.mkdir(exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    units = _units(BUILD)
    jobs = jobs or max(1, os.cpu_count() or 1)
    # biggest units first so the long poles start early
    order = sorted(units, key=lambda u: -int(next((d.split("=")[1] for d in u[2] if "PM_LG" in d), "0")))
    logs = []
    with ThreadPoolExecutor(jobs) as ex:
        for obj, log in ex.map(lambda u: _compile(u, force, verbose), order):
            if log:
                logs.append(f"== {obj.name}\n{log}")
    objs = [str(u[1]) for u in units]
    newest = max(Path(o).stat().st_mtime for o in objs)
    if force or not lib.exists() or lib.stat().st_mtime < newest:
        tmp = lib.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    if verbose and logs:
        (BUILD / "ptxas.log").write_text("\n".join(logs))
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--verbose", action="store_true", help="keep ptxas -v output in build/ptxas.log")
    ap.add_argument("--out", default=None, help="output .so path (default: lib/libphasemask_b200.so)")
    a = ap.parse_args(argv)
    print(build(a.force, a.jobs, a.verbose, a.out))


if __name__ == "__main__":
    sys.exit(main())
