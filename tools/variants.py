"""Build compile-time variants of libedgc_b200.so into alt_libs/ for A/B timing.

    python tools/variants.py name:-DEDGC_TD=0,-DEDGC_STCS=0 name2:...

Every source is recompiled with the extra defines.  Select a variant at run
time with EDGC_LIB_PATH.
"""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_10333_b200 import _build  # noqa: E402


def main():
    _build.build()
    objdir = os.path.join(_build.HERE, "_obj")
    out = os.path.join(ROOT, "alt_libs")
    os.makedirs(out, exist_ok=True)
    flags = _build.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                           "-I", os.path.join(ROOT, "include")]
    procs = []
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition(":")
        defs = [d for d in defs.split(",") if d]
        objs = []
        for src in _build.sources():
            obj = os.path.join(out, f"{name}_{os.path.basename(src).replace('.cu', '.o')}")
            objs.append(obj)
            procs.append((name, subprocess.Popen([_build.NVCC] + flags + defs + ["-c", src, "-o", obj])))
        procs.append((name, objs))
    pending = {}
    for name, p in procs:
        if isinstance(p, list):
            pending[name] = p
            continue
        if p.wait() != 0:
            raise SystemExit(f"variant {name} failed")
    for name, objs in pending.items():
        lib = os.path.join(out, f"{name}.so")
        subprocess.run([_build.NVCC] + _build.ARCH + ["-shared", "-o", lib] + objs + ["-cudart", "static"], check=True)
        print(lib)


if __name__ == "__main__":
    main()
