"""Build and time compile-time variants of one CUDA source (tuning experiments only).

    python tools/variants.py build NAME SRC.cu -DXL_FOO=1 ...   # here (nvcc cross-compiles)
    python tools/variants.py time NAME CFG PREC DROPS [REPS]     # on the GPU box

A variant is the product library with SRC's object recompiled with extra -D flags, linked
into _var/NAME/libxlmimo.so next to a copy of the binding, and imported under its own
module name.  The product build (paper_2503_18118_b200/) is untouched.
"""
import importlib.util
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PKG = os.path.join(ROOT, "paper_2503_18118_b200")


def build(name, src, flags):
    spec = importlib.util.spec_from_file_location("_xl_build", os.path.join(PKG, "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()
    out = os.path.join(ROOT, "_var", name)
    os.makedirs(out, exist_ok=True)
    objs = []
    for s in b._sources():
        o = os.path.join(b.BUILD, os.path.basename(s) + ".o")
        if os.path.basename(s) == os.path.basename(src):
            o = os.path.join(out, os.path.basename(s) + ".o")
            subprocess.check_call([b.NVCC, *b.ARCH, *b.FLAGS, *flags, "-c", src, "-o", o])
        objs.append(o)
    subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-o", os.path.join(out, "libxlmimo.so"),
                           *objs])
    shutil.copy(os.path.join(PKG, "__init__.py"), os.path.join(out, "__init__.py"))
    shutil.copy(os.path.join(PKG, "parallel.py"), os.path.join(out, "parallel.py"))
    print("built", out)


def load(name):
    d = os.path.join(ROOT, "_var", name) if name != "product" else PKG
    spec = importlib.util.spec_from_file_location(f"xlv_{name}", os.path.join(d, "__init__.py"),
                                                  submodule_search_locations=[d])
    m = importlib.util.module_from_spec(spec)
    sys.modules[f"xlv_{name}"] = m
    spec.loader.exec_module(m)
    return m


def time_variant(name, cfg, prec, drops, reps=5):
    import statistics
    import torch
    from workloads import CONFIGS
    xl = load(name)
    w = CONFIGS[cfg]
    arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, drops, seed=w.seed)
    p = {"fp64": xl.FP64, "fp32": xl.FP32, "mat32": xl.FP32}[prec]
    mode = xl.MATERIALIZED if prec == "mat32" else xl.FUSED
    G = xl.gram_exact(arr, pos, precision=p, mode=mode)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        G = xl.gram_exact(arr, pos, precision=p, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:24s} cfg{cfg} {prec} D={drops}: {statistics.median(ts):.3f} ms  G00={float(G[0,0,0].real):.6e}",
          flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3], sys.argv[4:])
    else:
        time_variant(sys.argv[2], int(sys.argv[3]), sys.argv[4], int(sys.argv[5]),
                     int(sys.argv[6]) if len(sys.argv) > 6 else 5)
