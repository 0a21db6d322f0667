"""Summarise tools/gemm_trace.py output: per-k-block MMA interval, per-tile
mainloop and epilogue (tfull -> release -> done) cycles."""
import statistics
import sys

for f in sys.argv[1:]:
    L = open(f).read().splitlines()
    print(L[0])
    ev = [(int(l.split()[0]), int(l.split()[2]), l.split()[3]) for l in L[1:]]
    fulls = [t for t, u, n in ev if n == "M.full"]
    d = [b - a for a, b in zip(fulls, fulls[1:])]
    print(f"  M.full interval median {statistics.median(d)} mean {sum(d) / len(d):.0f} max {max(d)}")
    for u in sorted(set(u for _, u, _ in ev))[:8]:
        e = {n: t for t, uu, n in ev if uu == u and n != "M.full"}
        fl = [t for t, uu, n in ev if uu == u and n == "M.full"]
        print(f"  unit {u:4d}: main {e.get('M.commit', 0) - fl[0]:6d}  epi tfull->release "
              f"{e.get('E.release', 0) - e.get('E.tfull', 0):5d} ->done {e.get('E.done', 0) - e.get('E.tfull', 0):5d}"
              f"  acc wait {e.get('M.accfree', 0) - e.get('M.tile', 0):5d}  first-load {fl[0] - e.get('P.stage0', 0):5d}")
    print(f"  span {max(t for t, _, _ in ev) - min(t for t, _, _ in ev)} cycles")
