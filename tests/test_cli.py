"""SPEC cli `validate` on the shipped scenarios (CPU)."""
import glob
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.usefixtures("built")


@pytest.mark.parametrize("sc", sorted(glob.glob(os.path.join(ROOT, "scenarios", "*.json"))))
def test_validate_scenarios(sc):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "opflow_cli.py"), "validate",
                        "--config", sc], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
