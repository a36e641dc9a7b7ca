"""Build libkmb.so variants with -D flags into variants/ (A/B experiments;
select one at run time with KMB_LIB=variants/libkmb_<name>.so)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_01182_b200 import _build as B
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)

def one(spec):
    name, defs = spec.split("=", 1) if "=" in spec else (spec, "")
    out = os.path.join(ROOT, "variants", f"libkmb_{name}.so")
    srcs = [os.path.join(B.CSRC, s) for s in B.CU_SOURCES]
    cmd = [B.NVCC, *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-I", B.INCLUDE, "-I", B.CSRC, *[f"-D{d}" for d in defs.split(",") if d], *srcs,
           "-o", out, "-lcudart", "-ldl"]
    subprocess.run(cmd, check=True)
    return out

with ThreadPoolExecutor(8) as ex:
    for o in ex.map(one, sys.argv[1:]):
        print(o)
