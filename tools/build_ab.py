"""Build an A/B variant of the product library with ONE kernel source taken
from a git revision (everything else from the working tree), for same-box
timing comparisons: OPF_LIB=<out> python tools/gemm_ab.py.
Usage: python tools/build_ab.py <rev> <csrc-relative .cu path> <out.so> [stub.cu]
(e.g. c235f36 kernels/gemm.cu paper_2605_21603_b200/libopflow_b200_gemm_r0.so tools/ab_stubs/splitk_stub.cu)"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_21603_b200 import build as B  # noqa: E402

rev, rel, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
extra = sys.argv[4:]
tmp = ROOT / "paper_2605_21603_b200" / "_build" / "ab"
tmp.mkdir(parents=True, exist_ok=True)
src = tmp / Path(rel).name
if rev.startswith("file:"):  # a patched copy of the source instead of a git revision
    src.write_text(Path(rev[5:]).read_text())
else:
    src.write_text(subprocess.run(["git", "-C", str(ROOT), "show", f"{rev}:paper_2605_21603_b200/csrc/{rel}"],
                                  capture_output=True, text=True, check=True).stdout)
B.build()
objs = []
for o in sorted(B.OBJ.glob("*.o")):
    if o.name == Path(rel).parent.name + "_" + Path(rel).name + ".o":
        continue
    objs.append(str(o))
for s in [src] + [Path(e) for e in extra]:
    o = tmp / (s.name + ".o")
    subprocess.run([B.NVCC, *B.NVFLAGS, *B.INCLUDES, "-c", str(s), "-o", str(o)], check=True)
    objs.append(str(o))
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(out), *objs, "-cudart", "static",
                "-ldl", "-lpthread", f"-Xlinker=--version-script={B.CSRC / 'exports.map'}", "-Xlinker=-Bsymbolic"],
               check=True)
print(out)
