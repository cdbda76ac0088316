"""Per-CUDA-line instruction/stall breakdown of one kernel in an ncu report (dev aid).
usage: ncu_lines.py REPORT KERNEL_REGEX [N]"""
import collections, csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(r for r in rows if r and r[0] == "Line No")
ii = h.index("Instructions Executed"); wi = h.index("Warp Stall Sampling (All Samples)")
cur = None; seen = set(); acc = collections.Counter(); st = collections.Counter(); src = {}
curfile = ""
for r in rows:
    if r and r[0] == "File Path":
        curfile = r[1].split("/")[-1]
    if len(r) > ii and r[0] not in ("", "Line No") and r[2] == "-":
        cur = (curfile, r[0]); src[cur] = r[1].strip()[:90]
    elif len(r) > ii and r[0] == "" and r[2].startswith("0x"):
        if r[2] in seen:
            continue
        seen.add(r[2])
        try:
            acc[cur] += int(r[ii]); st[cur] += int(r[wi])
        except ValueError:
            pass
tot = sum(acc.values()); ts = sum(st.values()) or 1
print("total warp inst", tot)
for k, v in sorted(acc.items(), key=lambda kv: -(kv[1] / tot + st[kv[0]] / ts))[:N]:
    print(f"{v/tot:.3f} st={st[k]/ts:.3f} {k[0]}:{k[1]} {src.get(k,'')}")
