"""The C-ABI boundary (CPU): the in-tree library loads, exports exactly the
functions include/opflow_b200.h declares, the header compiles as plain C, and
a C program can drive the frontend through it (the reference-side FFI of
INTEGRATION.md)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "opflow_b200.h")
LIB = os.path.join(ROOT, "paper_2605_21603_b200", "libopflow_b200.so")
pytestmark = pytest.mark.usefixtures("built")


def declared():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(opf_[a-z_0-9]+)\s*\(", text)) - {"opf_kernel_fn", "opf_schedule_fn", "opf_status"})


def test_library_exports_every_declared_symbol():
    names = declared()
    assert len(names) >= 45
    lib = ctypes.CDLL(LIB)
    for n in names:
        assert hasattr(lib, n), n
    exported = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    dyn = {l.split()[-1] for l in exported.splitlines() if " T " in l}
    assert set(names) <= dyn
    assert all(s.startswith("opf_") for s in dyn), sorted(s for s in dyn if not s.startswith("opf_"))[:5]


C_PROGRAM = r"""
#include <stdio.h>
#include <string.h>
#include "opflow_b200.h"
int main(void) {
  const char* desc =
    "{\"tensors\":[{\"name\":\"x\",\"shape\":[4,4],\"role\":\"input\"},"
    "{\"name\":\"w\",\"shape\":[4,4],\"batch\":\"replicated\",\"role\":\"weight\"},"
    "{\"name\":\"m\",\"shape\":[4,4]},{\"name\":\"y\",\"shape\":[4,4],\"role\":\"output\"}],"
    "\"operators\":[{\"name\":\"mm\",\"kind\":\"MatMul\",\"inputs\":[\"x\",\"w\"],\"outputs\":[\"m\"]},"
    "{\"name\":\"ar\",\"kind\":\"AllReduce\",\"inputs\":[\"m\"],\"outputs\":[\"y\"],\"attrs\":{\"world_size\":2}}]}";
  opf_graph* g = 0; opf_plan* p = 0; char* dump = 0;
  if (opf_graph_build(desc, &g)) { printf("build: %s\n", opf_last_error()); return 1; }
  if (opf_partition(g, "[{\"kind\":\"func\",\"pattern\":\"AllReduce\"}]", &p)) return 2;
  if (opf_validate_plan(p, g)) return 3;
  if (opf_plan_dump(p, &dump)) return 4;
  int ok = strstr(dump, "\"label\":\"ar\"") != 0;
  opf_free_string(dump);
  /* the error contract: Errc ordinal + 1, message via opf_last_error */
  opf_graph* bad = 0;
  opf_status st = opf_graph_build("{\"tensors\":[],\"operators\":[{\"name\":\"o\",\"kind\":\"ElemAdd\","
                                  "\"inputs\":[\"a\"],\"outputs\":[\"b\"]}]}", &bad);
  printf("%s %d %s\n", ok ? "OK" : "BAD", st, opf_errc_name(st));
  opf_plan_free(p); opf_graph_free(g);
  return ok ? 0 : 5;
}
"""


def test_c_program_drives_the_abi(tmp_path):
    src = tmp_path / "abi_client.c"
    src.write_text(C_PROGRAM)
    exe = tmp_path / "abi_client"
    libdir = os.path.dirname(LIB)
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", str(src), "-I", os.path.join(ROOT, "include"),
                        "-L", libdir, "-lopflow_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    # unknown tensor 'a' -> Errc::UnknownTensor (ordinal 1) + 1 = 2
    assert r.stdout.strip() == "OK 2 UnknownTensor"
