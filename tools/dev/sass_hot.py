"""Per-source-line hot spots of one kernel from an ncu SASS source page (dev aid).

    python tools/dev/sass_hot.py <ncu_sass.csv> <nvdisasm -gi dump> <mangled-substring> [top]

The ncu csv is `ncu -i rep --page source --csv --print-source sass -k NAME`;
the dump is `nvdisasm -gi -c` of the cubin that was profiled.  Instruction
offsets are matched to the innermost .debug_line entry.
"""
import collections
import csv
import re
import sys

csv_path, dis_path, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
SRC = "/root/repo/paper_1111_3297_b200/csrc/sieve_kernels.cuh"
src_lines = open(SRC).read().split("\n")

# offset -> line for the function
off2line = {}
cur = None
inside = False
for ln in open(dis_path):
    if ln.startswith("\t.section") or ln.startswith(".section"):
        inside = ".text." in ln and fn in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*?", line (\d+)', ln)
    if m:
        cur = int(m.group(1))  # innermost line (inlined code keeps its own line)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur is not None:
        off2line[int(m.group(1), 16)] = cur

rows = list(csv.reader(open(csv_path)))
h = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[h]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
it = hdr.index("Thread Instructions Executed")
data = [r for r in rows[h + 1:] if len(r) > ie and r[ia].startswith("0x")]
a0 = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0, 0])
tot_i = tot_s = 0
for r in data:
    off = int(r[ia], 16) - a0
    line = off2line.get(off, -1)
    ins, smp, thr = int(r[ie] or 0), int(r[iss] or 0), int(r[it] or 0)
    agg[line][0] += ins
    agg[line][1] += smp
    agg[line][2] += thr
    tot_i += ins
    tot_s += smp
print(f"{fn}: {len(data)} SASS, {tot_i} warp-instr, {tot_s} stall samples, mapped {len(off2line)}")
for line, (ins, smp, thr) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    txt = src_lines[line - 1].strip()[:90] if line > 0 else "?"
    print(f"L{line:5d} instr {ins / tot_i:6.1%} samples {smp / max(tot_s, 1):6.1%} lanes {thr / max(ins, 1):5.1f} | {txt}")
