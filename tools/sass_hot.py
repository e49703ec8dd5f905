"""Summarise an ncu SASS source page: hottest instructions and stall samples, grouped in address windows."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie = hdr.index("Instructions Executed"); sm = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), r[1].strip(), float(r[ie]), float(r[sm])))
    except Exception:
        pass
tot_i = sum(d[2] for d in data); tot_s = sum(d[3] for d in data)
print("total inst", tot_i, "samples", tot_s)
# windows of 64 instructions
W = int(sys.argv[2]) if len(sys.argv) > 2 else 48
for i in range(0, len(data), W):
    blk = data[i:i + W]
    si = sum(d[2] for d in blk); ss = sum(d[3] for d in blk)
    if si / tot_i > 0.01 or ss / max(tot_s, 1) > 0.01:
        top = max(blk, key=lambda d: d[3])
        print("%5d %6.1f%% inst %6.1f%% samp  e.g. %s | hot: %s" % (i, 100 * si / tot_i, 100 * ss / max(tot_s, 1), blk[0][1][:40], top[1][:50]))
