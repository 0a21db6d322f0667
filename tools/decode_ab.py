"""Same-box A/B of the decode leg (BASELINE configs[3]) under environment
switches: each variant runs bench.run_decode in a fresh process (the kernels
read their switches once), interleaved over `--reps` rounds.
Usage: python tools/decode_ab.py --layers 8 --var base: --var ef_off:OPF_DECODE_L2=normal"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    import bench
    from paper_2605_21603_b200 import opflow as of
    bench.ROUNDS, bench.SOAK_S = 3, 1.0
    p = argparse.Namespace(layers=int(os.environ["AB_LAYERS"]), decode_batch=int(os.environ.get("AB_BATCH", 512)),
                           decode_ctx=int(os.environ.get("AB_CTX", 4096)), steps=5,
                           warmup=3, rounds=3, soak=1.0,
                           sm_sweep=[int(x) for x in os.environ.get("AB_SMS", "").split()] or [])
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    r = bench.run_decode(of, torch, dev, p, 1, None, 0, 1, stream)
    print("RESULT " + json.dumps({"strategies_ms": r["strategies_ms"], "attn_gbs": r["roofline"]["achieved"]}))
    sys.exit(0)

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--sms", default="40")
ap.add_argument("--var", action="append", required=True, help="name:K=V,K=V")
a = ap.parse_args()
out = {}
for rep in range(a.reps):
    for v in a.var:
        name, _, kv = v.partition(":")
        env = dict(os.environ, AB_LAYERS=str(a.layers), AB_SMS=a.sms.replace(",", " "))
        for item in filter(None, kv.split(",")):
            k, _, val = item.partition("=")
            env[k] = val
        res = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        line = [l for l in res.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(name, "FAILED", res.stderr[-2000:])
            continue
        r = json.loads(line[0][7:])
        out.setdefault(name, []).append(r)
        print(name, rep, json.dumps(r), flush=True)
print("SUMMARY " + json.dumps(out))
