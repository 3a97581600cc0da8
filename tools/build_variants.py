#!/usr/bin/env python
"""Build libfbp.so variants that differ in compile-time switches (A/B
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
    jobs = [(v, src) for v in variants for src in srcs]
    with cf.ThreadPoolExecutor(12) as ex:
        objs = list(ex.map(lambda j: cc(j[1], os.path.join(OUT, f"{j[0][0]}_{os.path.basename(j[1])}.o"), j[0][1]),
                           jobs))
    for name, _ in variants:
        mine = [o for (v, _), o in zip(jobs, objs) if v[0] == name]
        so = os.path.join(OUT, f"{name}.so")
        r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", so] + mine +
                           ["-lcudart_static", "-lrt", "-ldl", "-lpthread"], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        print(so)
    for o in objs:
        os.remove(o)


if __name__ == "__main__":
    main()
