"""ncu source page (SASS) of kernel #k in a report -> top stall lines mapped to CUDA source lines via nvdisasm -g."""
import csv, io, re, subprocess, sys, collections
rep, kidx, cubin, fn = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
ks = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
start = ks[kidx]; end = ks[kidx + 1] if kidx + 1 < len(ks) else len(rows)
h = rows[start + 1]
si = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[start + 2:end] if len(r) > si]
base = int(data[0][0], 16)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
s0 = [i for i, l in enumerate(dis) if l.startswith(".text." + fn + ":")][0]
a2l, cur = {}, None
for l in dis[s0 + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
tot = sum(float(r[si] or 0) for r in data)
byline = collections.Counter()
for r in data:
    byline[a2l.get(int(r[0], 16) - base, ("?", 0))] += float(r[si] or 0)
print("samples", tot)
for (f, ln), v in byline.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 25):
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}")
