"""TEST INFRASTRUCTURE — writes the graph descriptions the CPU reference arm
evaluates (bench.py --impl reference / cpu_baseline), so that arm never loads
the product library: Llama-3-8B-shaped single layers (fp32, TP=1, one
sequence of `rows` tokens) and BASELINE configs[0]'s toy decoder.

The descriptions come from the product's builders (csrc/host/builders.cpp);
tests/test_fixtures.py pins the committed files to them.

    python oracle/fixtures/make_fixtures.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
LLAMA = dict(hidden=4096, heads=32, kv_heads=8, head_dim=128, inter=14336)
REF_ROWS = (64, 128)


def expected() -> dict:
    sys.path.insert(0, str(ROOT))
    from paper_2605_21603_b200 import opflow as of
    out = {f"llama3_8b_layer_f32_rows{r}.json": of.llama_graph(layers=1, tokens=r, seq_len=r, tp=1, dtype="f32",
                                                                **LLAMA)
           for r in REF_ROWS}
    out["toy_decoder_c1.json"] = of.toy_decoder_graph()
    return {k: json.dumps(json.loads(v), sort_keys=True) for k, v in out.items()}


def load(name: str) -> str:
    return (HERE / name).read_text()


if __name__ == "__main__":
    for name, text in expected().items():
        (HERE / name).write_text(text + "\n")
        print(name, len(text))
