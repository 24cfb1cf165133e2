"""Build libpqb200.so (the sm_100a C-ABI library) in-tree with nvcc.

    python -m paper_2502_00527_b200.build [--verbose-ptxas] [--force]

Each .cu is compiled to an object in build/ (re-used when its sources are
unchanged), then linked with the static CUDA runtime into
paper_2502_00527_b200/libpqb200.so, so the library travels with the repo
snapshot and needs only the driver at run time.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "pqb200"
LIB = PKG / "libpqb200.so"
SOURCES = ["encode.cu", "encode_fast.cu", "decode.cu", "decode_dq.cu", "decode_dq_lin.cu", "misc.cu", "api.cu", "abi.cu"]
# .cu files a source #includes (their text is part of its digest)
INCLUDES = {"decode_dq_lin.cu": ["decode_dq.cu"]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC,-O2,-Wall",
    "-Xptxas",
    "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (set NVCC or add /usr/local/cuda/bin to PATH)")


def _digest(src: Path, extra: list[str]) -> str:
    h = hashlib.sha256()
    h.update(" ".join(extra).encode())
    deps = [CSRC / n for n in INCLUDES.get(src.name, [])]
    for p in sorted(list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "pqb200.h", src] + deps):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def _gen_tables() -> None:
    subprocess.run([sys.executable, str(CSRC / "gen_tables.py"), str(CSRC / "angle_tables.h")], check=True)


def build(force: bool = False, verbose_ptxas: bool = False, jobs: int | None = None,
          defines: tuple[str, ...] = (), out: Path | None = None) -> Path:
    """Compile + link libpqb200.so.  defines / out build an A/B variant of the
    library elsewhere (e.g. build_ab/) without touching the in-tree one."""
    _gen_tables()
    BUILD.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    flags = ARCH + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose_ptxas else []) + [f"-D{d}" for d in defines]
    lib = Path(out) if out is not None else LIB
    objs: list[Path] = []
    todo: list[tuple[Path, Path, Path]] = []
    for name in SOURCES:
        src = CSRC / name
        tag = _digest(src, flags)
        obj = BUILD / f"{src.stem}.{tag}.o"
        objs.append(obj)
        if force or not obj.exists():
            todo.append((src, obj, BUILD / f"{src.stem}.log"))

    def compile_one(item: tuple[Path, Path, Path]) -> tuple[Path, int, str]:
        src, obj, log = item
        cmd = [cc, *flags, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log.write_text(res.stdout + res.stderr)
        return src, res.returncode, res.stdout + res.stderr

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or min(len(todo), os.cpu_count() or 4)) as ex:
            for src, rc, out in ex.map(compile_one, todo):
                if rc != 0:
                    raise RuntimeError(f"nvcc failed on {src.name}:\n{out}")
                if verbose_ptxas:
                    print(out)
    # relink when any object is new or the lib was linked from another object set
    # (switching back to an older source version reuses its cached objects,
    # which are older than the lib built in between)
    stamp = lib.with_suffix(".so.objs")
    obj_set = "\n".join(o.name for o in objs)
    if (force or todo or not lib.exists() or not stamp.exists() or stamp.read_text() != obj_set
            or any(o.stat().st_mtime > lib.stat().st_mtime for o in objs)):
        lib.parent.mkdir(parents=True, exist_ok=True)
        tmp = lib.with_suffix(".so.tmp")
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}{res.stderr}")
        os.replace(tmp, lib)
        stamp.write_text(obj_set)
    if out is None:  # drop stale objects of older source versions
        keep = {o.name for o in objs}
        for o in BUILD.glob("*.o"):
            if o.name not in keep:
                o.unlink()
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose-ptxas", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose_ptxas=args.verbose_ptxas))


if __name__ == "__main__":
    main()
