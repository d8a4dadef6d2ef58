"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel totals and shares.  usage: launch_summary.py LAUNCHES_CSV OUT_JSON"""
import csv, io, json, re, sys

src, dst = sys.argv[1], sys.argv[2]
txt = open(src).read().split("\n")
i = next(k for k, l in enumerate(txt) if l.startswith('"ID"'))
agg = {}
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void ", "", r["Kernel Name"]).split("<")[0].split("(")[0].replace("gfq::", "")
    ms = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    a = agg.setdefault(name, [0.0, 0])
    a[0] += ms
    a[1] += 1
tot = sum(a[0] for a in agg.values())
out = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none on `python bench.py --steps 1 "
                 "--warmup 0 --no-e2e --no-cpu --no-convergence` (C5, 8192 frames, 50 iterations, PUS+SUS): "
                 "cold-cache, serialised per-launch device times",
       "total_ms": round(tot, 1),
       "kernels": {k: {"ms": round(v[0], 3), "launches": v[1], "share": round(v[0] / tot, 4)}
                   for k, v in sorted(agg.items(), key=lambda x: -x[1][0])}}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out)[:700])
