#!/usr/bin/env python
"""Build libfbp.so variants that differ in sweep.cu compile-time switches (A/B
measurement on one GPU call).  Output: paper_2007_06289_b200/variants/<name>.so.

    python tools/build_variants.py name1:-DFOO=1,-DBAR=0 name2:-DFOO=0 ...

On the GPU box: cp paper_2007_06289_b200/variants/<name>.so paper_2007_06289_b200/libfbp.so
before each measurement (the binding loads libfbp.so; nothing rebuilds it at run time).
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_06289_b200 import build as B  # noqa: E402

OUT = os.path.join(B.PKG, "variants")


def cc(src, obj, extra):
    cmd = [B.NVCC] + B.ARCH + B.FLAGS + extra + ["-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return obj


def main():
    os.makedirs(OUT, exist_ok=True)
    variants = [(a.split(":")[0], [f for f in a.split(":")[1].split(",") if f]) for a in sys.argv[1:]]
    srcs = B.sources()
    sweep = [s for s in srcs if s.endswith("sweep.cu")][0]
    others = [s for s in srcs if s != sweep]
    with cf.ThreadPoolExecutor(8) as ex:
        common = list(ex.map(lambda s: cc(s, os.path.join(OUT, os.path.basename(s) + ".o"), []), others))
        vobj = list(ex.map(lambda v: cc(sweep, os.path.join(OUT, f"sweep_{v[0]}.o"), v[1]), variants))
    for (name, _), o in zip(variants, vobj):
        so = os.path.join(OUT, f"{name}.so")
        r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", so, o] + common +
                           ["-lcudart_static", "-lrt", "-ldl", "-lpthread"], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        print(so)
    for o in common + vobj:
        os.remove(o)


if __name__ == "__main__":
    main()
