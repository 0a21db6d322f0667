"""Fit the context-aware strategy selector on the bench's
Llama-3-8B prefill graph and check its predictions.

Binds max-size buffers once and runs row-prefix views at each calibration batch
(one cached plan + CUDA graph per (strategy, rows)), fits alpha + beta * rows per
candidate (`paper_2605_21603_b200/selector.py`), then replays the fitted
decision table at held-out batch sizes and compares predicted vs measured ms.

  python tools/calibrate_selector.py --layers 4 --out gpurun_out/selector_prefill.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--max-tokens", type=int, default=8192)
    ap.add_argument("--seq-len", type=int, default=1024)
    ap.add_argument("--points", default="1024,2048,4096,8192")
    ap.add_argument("--holdout", default="3072,6144")
    ap.add_argument("--margin", type=float, default=0.01)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2605_21603_b200 import opflow as of
    from paper_2605_21603_b200 import selector as sl

    dev = torch.device("cuda", 0)
    T, S = a.max_tokens, a.seq_len
    desc = of.llama_graph(layers=a.layers, tokens=T, seq_len=S, dtype="bf16", **bench.LLAMA)
    g, plan, sess, bufs = bench.build_session(of, desc, [], dev, None, seed=7)
    bufs["positions"] = (torch.arange(T, device=dev) % S).to(torch.int64)
    batched = {t["name"] for t in g.description["tensors"]
               if t.get("batch", "batched") == "batched" and t["name"] in bufs}

    def bind_rows(r):
        for n in batched:
            sess.bind(n, bufs[n][:r])
        return sess

    cands = [{"name": "sequential"},
             {"name": "split_overlap", "n_microbatches": 2, "align": S, "lane_mode": "ubatch"},
             {"name": "split_overlap", "n_microbatches": 2, "align": S}]
    # power soak so calibration runs at the capped clock the bench sees
    bind_rows(T)
    t_end = time.time() + 2.0
    while time.time() < t_end:
        sess.run(cands[0])
        torch.cuda.synchronize()
    pts = [int(x) for x in a.points.split(",")]
    sel = sl.calibrate(bind_rows, cands, pts, reps=3, rounds=3, margin=a.margin)
    rep = sel.report()
    spec = sel.spec()
    check = []
    for r in [int(x) for x in a.holdout.split(",")] + pts:
        s = bind_rows(r)
        meas = {json.dumps(c, sort_keys=True): sl.time_forward(s, c, reps=3) for c in cands}
        table_ms = sl.time_forward(s, spec, reps=3)
        pick = sel.choose(r)
        best = min(meas, key=meas.get)
        check.append({"rows": r, "pick": pick, "table_ms": table_ms,
                      "predicted_ms": {k: sel.predict(json.loads(k), r) for k in meas},
                      "measured_ms": meas, "measured_best": json.loads(best),
                      "pick_regret": meas[json.dumps(pick, sort_keys=True)] / meas[best] - 1.0})
    out = {"workload": f"llama3-8b prefill, {a.layers} layers, seq_len {S}, rows <= {T}, bf16",
           "gpu": torch.cuda.get_device_name(0), "selector": rep, "engine_spec": spec, "check": check}
    text = json.dumps(out, indent=1)
    print(text)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
