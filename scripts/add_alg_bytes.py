"""Add the algorithmic bytes of the captured launches to profiles/<dir>/ncu_traffic_<cfg>.json
(8q bytes per edge-message update; a SUS level of e edges is 2e updates per frame)
so that bench.py can report roofline.traffic = ncu DRAM bytes per algorithmic byte x its own launch.
usage: add_alg_bytes.py JSON CONFIG FRAMES SUS_LEVEL(1-based) PUS_WAVE_FRAMES"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth

path, name, frames, lvl, wave = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
cfg = synth.CONFIGS[name]
code = synth.code_for(cfg)
rows = np.concatenate([code.A_row, code.B_row]); cols = np.concatenate([code.A_col, code.B_col + code.N])
V = code.N + code.M
by_col = [[] for _ in range(V)]
for r, c in zip(rows.tolist(), cols.tolist()):
    by_col[c].append(r)
rowlvl = np.zeros(code.M, dtype=np.int64); level = np.zeros(V, dtype=np.int64)
for j in range(V):                      # index order (A7): DESIGN.md §5
    L = 1 + max((rowlvl[i] for i in by_col[j]), default=0)
    level[j] = L
    for i in by_col[j]:
        rowlvl[i] = L
edges = sum(len(by_col[j]) for j in range(V) if level[j] == lvl)
d = json.load(open(path))
q, E = cfg.q, len(rows)
for k, v in d["kernels"].items():
    if k == "sus":
        alg = 8.0 * q * 2 * edges * frames
        v["note"] = "captured launch = SUS level %d of %d (%d edges) over %d frames; algorithmic bytes 8q x 2 x %d x %d" % (
            lvl, int(level.max()), edges, frames, edges, frames)
    else:
        alg = 8.0 * q * E * wave
        v["note"] = "captured launch = first PUS wave (%d frames); algorithmic bytes 8q x E x %d" % (wave, wave)
    v["alg_bytes_this_launch"] = alg
    v["dram_per_alg_byte"] = v["dram_bytes_per_launch"] / alg
    print(k, v["note"], round(v["dram_per_alg_byte"], 4))
json.dump(d, open(path, "w"), indent=1)
