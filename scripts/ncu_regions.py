"""Warp instructions and shared-memory wavefronts per code region of one ncu source page (csv):
    ncu -i rep --page source --csv > src.csv; python scripts/ncu_regions.py src.csv "[(name, first_offset, end_offset), ...]"
Offsets are SASS addresses relative to the kernel start (cuobjdump -sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia = hdr.index("Instructions Executed"); isrc = hdr.index("Source"); iad = hdr.index("Address")
iw = hdr.index("L1 Wavefronts Shared"); ismp = hdr.index("# Samples")
data = rows[2:]
base = int(data[0][iad], 16)
tot = sum(int(r[ia]) for r in data)
totw = sum(int(r[iw]) for r in data)
print("total warp inst %.4g  smem wavefronts %.4g" % (tot, totw))
# regions by address offset
regions = eval(sys.argv[2]) if len(sys.argv) > 2 else []
for name, a, b in regions:
    s = sum(int(r[ia]) for r in data if a <= int(r[iad],16)-base < b)
    w = sum(int(r[iw]) for r in data if a <= int(r[iad],16)-base < b)
    smp = sum(int(r[ismp]) for r in data if a <= int(r[iad],16)-base < b)
    print("%-28s inst %.4g (%.1f%%)  wavefronts %.4g (%.1f%%) samples %d" % (name, s, 100*s/tot, w, 100*w/max(totw,1), smp))
