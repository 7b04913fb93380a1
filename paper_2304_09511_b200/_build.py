"""In-tree build of libspmv_b200.so (sm_100a) with nvcc.

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (a JIT cache under ~/.cache would not).  Objects are
rebuilt only when a source or header is newer than the library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
OBJ_DIR = PKG_DIR / "_objs"
LIB_PATH = PKG_DIR / "libspmv_b200.so"
INCLUDE = REPO / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
    f"-I{INCLUDE}",
] + os.environ.get("SPMV_NVCC_EXTRA", "").split()


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool, obj_dir: Path = OBJ_DIR, flags=None) -> Path:
    obj = obj_dir / (src.stem + ".o")
    if not _stale(obj, [src, *_headers(), Path(__file__)]):
        return obj
    cmd = [NVCC, *(flags or NVCC_FLAGS), "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr.strip():
        print(res.stderr, file=sys.stderr)
    return obj


DEBUG_LIB_PATH = PKG_DIR / "libspmv_b200_debug.so"


def build(verbose: bool = False, force: bool = False, debug: bool = False) -> Path:
    """Compile every csrc/*.cu for sm_100a and link libspmv_b200.so.

    debug=True builds libspmv_b200_debug.so instead, with the device-side
    consistency checks (-DSPMV_DEBUG_CHECKS: TMA stages compared with global
    memory, panel indices bounds-checked; read with spmv_debug_check_counts)
    — the substitute for compute-sanitizer, which is closed on this pool.
    Select it at run time with SPMV_B200_LIB."""
    obj_dir = PKG_DIR / "_objs_debug" if debug else OBJ_DIR
    lib_path = DEBUG_LIB_PATH if debug else LIB_PATH
    nvcc_flags = NVCC_FLAGS + (["-DSPMV_DEBUG_CHECKS"] if debug else [])
    obj_dir.mkdir(exist_ok=True)
    srcs = _sources()
    stamp = obj_dir / "flags.txt"  # objects built with other flags are stale
    flags = " ".join(nvcc_flags)
    if not stamp.exists() or stamp.read_text() != flags:
        force = True
    if force:
        for o in obj_dir.glob("*.o"):
            o.unlink()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, obj_dir, nvcc_flags), srcs))
    stamp.write_text(flags)
    if force or _stale(lib_path, objs):
        # Export only the C ABI (spmv_*); static cudart and C++ internals stay local.
        cmd = [NVCC, *ARCH, "-shared", "-o", str(lib_path), *map(str, objs),
               "-Xlinker", f"--version-script={PKG_DIR / 'csrc' / 'exports.map'}"]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return lib_path


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv, debug="--debug" in sys.argv))
