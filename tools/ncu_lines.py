"""Aggregate `ncu --page source --print-source cuda,sass --csv` stall samples by CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 1
out, hdr, kernels = [], None, 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r; kernels += 1
        continue
    if kernels != which or not hdr or not r or r[0] in ("", "File Path", "Function Name"):
        continue
    try:
        out.append((int(r[hdr.index("# Samples")]), int(r[0]), int(r[hdr.index("Instructions Executed")]), r[1][:100]))
    except Exception:
        pass
tot = sum(o[0] for o in out)
print("total samples", tot)
for s, l, i, src in sorted(out, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 22]:
    print(f"{s:5d} {100*s/max(tot,1):5.1f}%  L{l:4d} inst={i:8d} {src}")
