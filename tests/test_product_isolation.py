"""CPU: the product path never routes through the oracle, and has no CPU fallback.

* No module or source file of the package (`paper_2605_21603_b200/`) imports,
  links or dlopens anything under `oracle/` (the CPU restatement and the
  compiled reference are test infrastructure only).
* The built library's dynamic dependencies do not include the reference build.
* With the CUDA library missing the package's device entry point raises
  instead of falling back to a host path."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2605_21603_b200"
ORACLE_REF = re.compile(r"\bimport\s+oracle\b|\bfrom\s+oracle\b|libopflow_ref|oracle/_ref|ref_shim|kernels_scalar")


def _sources():
    for p in PKG.rglob("*"):
        if p.suffix in (".py", ".cu", ".cpp", ".hpp", ".cuh", ".h") and "_build" not in p.parts:
            yield p


def test_package_sources_never_reference_the_oracle():
    hits = []
    for p in _sources():
        for i, line in enumerate(p.read_text(errors="replace").splitlines(), 1):
            code = line.split("//")[0] if p.suffix != ".py" else line.split("#")[0]
            if ORACLE_REF.search(code):
                hits.append(f"{p.relative_to(ROOT)}:{i}: {line.strip()}")
    assert not hits, "\n".join(hits)


def test_library_does_not_link_the_reference_build():
    so = PKG / "libopflow_b200.so"
    if not so.exists():
        pytest.skip("library not built")
    out = subprocess.run(["readelf", "-d", str(so)], capture_output=True, text=True).stdout
    needed = re.findall(r"\(NEEDED\).*\[(.*)\]", out)
    assert needed, out[:500]
    assert not [n for n in needed if "opflow_ref" in n or "oracle" in n], needed


def test_missing_library_fails_loudly(tmp_path):
    code = (
        "import sys, pathlib\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "import paper_2605_21603_b200._lib as L\n"
        f"L.LIB_PATH = pathlib.Path({str(tmp_path / 'absent.so')!r})\n"
        "L._lib = None\n"
        "try:\n"
        "    L.lib()\n"
        "except ImportError as e:\n"
        "    print('RAISED', 'no CPU fallback' in str(e))\n"
    )
    env = dict(os.environ)
    env.pop("OPF_LIB", None)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert "RAISED True" in r.stdout, r.stdout + r.stderr[-2000:]
