"""Export (function-relative address, executed count, stall samples, opcode) per SASS
instruction of the first kernel of an ncu report: sass_export.py REPORT OUT.csv"""
import csv, io, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Kernel Name"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[1]
print(hdr)
ii = hdr.index("Instructions Executed"); si = hdr.index("Source"); ws = hdr.index("Warp Stall Sampling (All Samples)")
ai = hdr.index("Address") if "Address" in hdr else None
with open(out, "w") as fh:
    w = csv.writer(fh)
    for n, r in enumerate(rows[2:]):
        if len(r) <= ws: continue
        w.writerow([r[ai] if ai is not None else n, r[ii], r[ws], r[si].strip()[:60]])
