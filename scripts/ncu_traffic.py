"""Summarise ncu --set full reports into profiles/<dir>/ncu_traffic.json:
per kernel: duration, dram bytes read+write per launch, throughput, occupancy, stall top-5.
usage: ncu_traffic.py OUT_JSON CONFIG REPORT [REPORT ...]"""
import csv, io, json, subprocess, sys

out_path, config, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
res = {"config": config, "kernels": {}}
units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tunits = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
for rep in reps:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, un = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, un))
        name = d["Kernel Name"].split("<")[0].split("(")[0].replace("void ", "").replace("gfq::", "")
        short = {"k_cn": "cn", "k_cn_dc": "cn", "k_big_cn": "cn", "k_vn": "vn", "k_big_vn": "vn", "k_sus": "sus",
                 "k_sus_dc": "sus", "k_sus_dc64": "sus", "k_big_sus": "sus"}.get(name, name)
        def num(k):
            try:
                return float(d[k])
            except Exception:
                return None
        rb = num("dram__bytes_read.sum") * units.get(u["dram__bytes_read.sum"], 1)
        wb = num("dram__bytes_write.sum") * units.get(u["dram__bytes_write.sum"], 1)
        dur = num("gpu__time_duration.sum") * tunits.get(u["gpu__time_duration.sum"], 1)
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        res["kernels"][short] = dict(
            report=rep, kernel=d["Kernel Name"][:120], duration_ms=dur,
            dram_bytes_per_launch=rb + wb, dram_read=rb, dram_write=wb,
            dram_gbs=(rb + wb) / (dur / 1e3) / 1e9,
            dram_pct_of_peak=num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            issue_active_pct=num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            fp64_pipe_pct=num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            warps_active_per_sm=num("sm__warps_active.avg.per_cycle_active"),
            registers=num("launch__registers_per_thread"),
            smem_per_block_kb=num("launch__shared_mem_per_block_dynamic"),
            top_stalls={n: round(v, 2) for v, n in stalls[:5]})
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
