"""Build a variant of the product library with ONE kernel source compiled
with extra nvcc flags (e.g. -DOPF_GEMM_TRACE), everything else from the
working tree: for same-box A/B timing or instrumentation.
Usage: python tools/build_variant.py <csrc-relative .cu> <out.so> <nvcc flag>...
(e.g. kernels/gemm.cu paper_2605_21603_b200/_build/libopflow_trace.so -DOPF_GEMM_TRACE)"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_21603_b200 import build as B  # noqa: E402

rel, out, flags = sys.argv[1], Path(sys.argv[2]), sys.argv[3:]
B.build()
src = B.CSRC / rel
tag = Path(rel).parent.name + "_" + Path(rel).name + ".o"
objs = [str(o) for o in sorted(B.OBJ.glob("*.o")) if o.name != tag]
vo = B.OBJ / "variant" / (out.stem + ".o")
vo.parent.mkdir(parents=True, exist_ok=True)
subprocess.run([B.NVCC, *B.NVFLAGS, *flags, *B.INCLUDES, "-c", str(src), "-o", str(vo)], check=True)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(out), *objs, str(vo), "-cudart", "static",
                "-ldl", "-lpthread", f"-Xlinker=--version-script={B.CSRC / 'exports.map'}", "-Xlinker=-Bsymbolic"],
               check=True)
print(out)
