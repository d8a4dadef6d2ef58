"""Build a tuning variant of libgfq.so: recompile ONE source with extra -D
defines and link it with the default objects of the others.
usage: python scripts/build_variant.py gfq_sus_dc.cu out.so -DGFQ_DC_S_MARKOV=3 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_cs_0605069_b200 import build as b  # noqa: E402

src, out, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()                                   # default objects up to date
tag = os.path.basename(out).replace(".so", "")
obj = os.path.join(b.CSRC, src.replace(".cu", "_" + tag + ".o"))
subprocess.check_call([b.NVCC, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj])
objs = [os.path.join(b.CSRC, s.replace(".cu", ".o")) for s in b.SOURCES if s != src] + [obj]
subprocess.check_call([b.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                       os.path.join(b.HERE, out), *objs, "-Xcompiler", "-fPIC"])
print(os.path.join(b.HERE, out))
