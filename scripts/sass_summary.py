"""Compact SASS summary of an ncu report (or its exported source-page CSV):
instruction mix and top stall lines.  usage: sass_summary.py REPORT|CSV"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
if rep.endswith(".csv"):          # an exported `--page source --csv --print-source sass`
    txt = open(rep).read()
else:
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    txt = subprocess.run(args, capture_output=True, text=True).stdout
lines = txt.splitlines()
# a report may hold several kernels: blocks start with "Kernel Name"
blocks, cur = [], []
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        if cur: blocks.append(cur)
        cur = [ln]
    else:
        cur.append(ln)
if cur: blocks.append(cur)
for b in blocks:
    rows = list(csv.reader(io.StringIO("\n".join(b))))
    print("==", rows[0][1][:100])
    hdr = rows[1]; data = rows[2:]
    ii = hdr.index("Instructions Executed"); si = hdr.index("Source"); ws = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter(); st = collections.Counter(); tot = 0; tots = 0; L = []
    for r in data:
        if len(r) <= ws: continue
        try: n = int(r[ii]); s = int(r[ws])
        except ValueError: continue
        src = r[si].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"): op = src.split()[1]
        op = op.split(".")[0]
        mix[op] += n; st[op] += s; tot += n; tots += s; L.append((s, n, src))
    print("total warp insts %.4g, stall samples %d" % (tot, tots))
    print(" ".join("%s:%.1f%%(st%.1f%%)" % (o, 100 * n / tot, 100 * st[o] / max(tots, 1)) for o, n in mix.most_common(22)))
    for s, n, src in sorted(L, reverse=True)[:25]:
        print("  %5.2f%% %11d  %s" % (100 * s / max(tots, 1), n, src[:90]))
