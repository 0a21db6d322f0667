"""Per-launch DRAM traffic of an `ncu --set full` capture of tools/profile_kernels.py
proj|proj_tp8 (two launches per shape, in the order that script runs them),
written as the JSON bench.py reads to fill roofline.traffic.
Usage: python tools/ncu_traffic.py OUT.json REP:shape1,shape2,... [REP:...]"""
import csv
import io
import json
import subprocess
import sys


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {k: h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                   "dram__bytes_write.sum")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
             "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
    res = []
    for r in rows[2:]:
        def val(k):
            i = col[k]
            return float(r[i].replace(",", "")) * scale.get(units[i], 1)
        res.append({"kernel": r[col["Kernel Name"]].split("(")[0], "us": val("gpu__time_duration.sum"),
                    "dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum")})
    return res


if __name__ == "__main__":
    table = {}
    for spec in sys.argv[2:]:
        rep, shapes = spec.split(":")
        ls = launches(rep)
        shapes = shapes.split(",")
        per = len(ls) // len(shapes)
        for i, s in enumerate(shapes):
            grp = ls[i * per:(i + 1) * per]
            table[s] = {"kernel": grp[0]["kernel"], "launches": len(grp),
                        "us": round(sum(x["us"] for x in grp) / len(grp), 2),
                        "dram_bytes": round(sum(x["dram_read"] + x["dram_write"] for x in grp) / len(grp)),
                        "source": rep.split("/")[-1]}
    json.dump(table, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(table, indent=1))
