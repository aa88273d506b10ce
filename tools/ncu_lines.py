"""Attribute an ncu SASS source page (CSV) to CUDA source lines via nvdisasm -g.

usage: python tools/ncu_lines.py <report.ncu-rep> <mangled-kernel-substring> [launch-block] [top]
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kname = sys.argv[1], sys.argv[2]
block_idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2204_07485_b200", "_lib", "libbigmeans_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if l.strip().startswith(".section") and kname in l)
lines, cur = {}, None
for l in dis[start + 1:]:
    if l.strip().startswith(".section") and ".text." in l:
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, curb = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        curb = [r]
        blocks.append(curb)
    elif curb is not None:
        curb.append(r)
b = blocks[block_idx]
print(b[0][1][:120])
hdr = b[1]
ia, isamp, iie = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [r for r in b[2:] if len(r) > isamp and r[ia].startswith("0x")]
base = min(int(r[ia], 16) for r in data)
per, ie = collections.Counter(), collections.Counter()
for r in data:
    key = lines.get(int(r[ia], 16) - base, ("?", 0))
    per[key] += int(r[isamp] or 0)
    ie[key] += int(r[iie] or 0)
tot, tie = sum(per.values()), sum(ie.values())
srcs = {}
print(f"samples {tot}  warp-instructions {tie}")
for (f, ln), v in sorted(per.items(), key=lambda x: -x[1])[:top]:
    path = os.path.join(ROOT, "paper_2204_07485_b200", "csrc", f)
    if f not in srcs:
        srcs[f] = open(path).read().split("\n") if os.path.exists(path) else []
    txt = srcs[f][ln - 1].strip()[:80] if 0 < ln <= len(srcs[f]) else ""
    print(f"{v:6d} {100 * v / tot:5.1f}%  ie {100 * ie[(f, ln)] / tie:5.1f}%  {f}:{ln}: {txt}")
