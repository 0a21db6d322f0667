"""Build the whole product library as of a git revision (temporary worktree)
into paper_2605_21603_b200/libopflow_b200_<rev>.so, for same-box A/B runs:
  OPF_LIB=paper_2605_21603_b200/libopflow_b200_<rev>.so python tools/gemm_ab.py
Usage: python tools/build_rev.py <rev>"""
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rev = sys.argv[1]
out = ROOT / "paper_2605_21603_b200" / f"libopflow_b200_{rev}.so"
with tempfile.TemporaryDirectory() as d:
    wt = Path(d) / "wt"
    subprocess.run(["git", "-C", str(ROOT), "worktree", "add", "--detach", str(wt), rev], check=True,
                   capture_output=True)
    try:
        subprocess.run([sys.executable, "-c", "from paper_2605_21603_b200.build import build; build()"], cwd=wt,
                       check=True)
        shutil.copy(wt / "paper_2605_21603_b200" / "libopflow_b200.so", out)
    finally:
        subprocess.run(["git", "-C", str(ROOT), "worktree", "remove", "--force", str(wt)], check=True)
print(out)
