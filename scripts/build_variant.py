"""Build an A/B variant of libvecattn.so with extra nvcc defines for one source file:
python scripts/build_variant.py <tag> <source.cu> -DFOO=1 ...  -> paper_2603_29494_b200/build/ab/lib_<tag>.so"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_29494_b200 import _build as b
tag, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()
out = os.path.join(b.BUILD, "ab")
os.makedirs(out, exist_ok=True)
obj = os.path.join(out, f"{tag}_{src.replace('.cu', '.o')}")
subprocess.check_call([b.NVCC, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj])
objs = [obj if s == src else os.path.join(b.BUILD, s.replace(".cu", ".o")) for s in b.SOURCES]
subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                       "-Xcompiler", "-fPIC", *objs, "-o", os.path.join(out, f"lib_{tag}.so")])
print(os.path.join(out, f"lib_{tag}.so"))
