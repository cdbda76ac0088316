#!/usr/bin/env python3
"""Per-source-line SASS breakdown of one kernel from an `ncu --set full
--import-source on` report: warp instructions, average active threads per
instruction (divergence), stall-sample share, and for shared-memory lines the
wavefronts against the ideal (bank conflicts).

    python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP] [--opcodes]
"""
import collections
import csv
import subprocess
import sys


def rows_of(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
    rows = rows_of(rep, kern)
    h = next(r for r in rows if r and r[0] == "Line No")
    col = {k: h.index(k) for k in ("Instructions Executed", "Thread Instructions Executed",
                                    "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared",
                                    "L1 Wavefronts Shared Ideal")}
    acc = collections.defaultdict(lambda: collections.Counter())
    ops = collections.Counter()
    src, cur, curfile, seen = {}, ("?", 0), "", set()
    for r in rows:
        if r and r[0] == "File Path":
            curfile = r[1].split("/")[-1]
        if len(r) > col["Instructions Executed"] and r[0] not in ("", "Line No") and r[2] == "-":
            cur = (curfile, int(r[0]))
            src[cur] = r[1].strip()[:80]
        elif len(r) > col["Instructions Executed"] and r[0] == "" and r[2].startswith("0x"):
            if r[2] in seen:
                continue
            seen.add(r[2])
            a = acc[cur]
            for k, i in col.items():
                a[k] += num(r[i])
            opc = r[3].split()[0] if r[3].split() else "?"
            if opc.startswith("@"):
                opc = r[3].split()[1] if len(r[3].split()) > 1 else opc
            ops[opc.split(".")[0]] += num(r[col["Instructions Executed"]])
    tot = sum(a["Instructions Executed"] for a in acc.values()) or 1
    ts = sum(a["Warp Stall Sampling (All Samples)"] for a in acc.values()) or 1
    print(f"# {kern}: {tot:.0f} warp instructions")
    print("inst%  stall%  thr/inst  smem_wf/ideal  line  source")
    key = lambda kv: -(kv[1]["Instructions Executed"] / tot + kv[1]["Warp Stall Sampling (All Samples)"] / ts)
    for k, a in sorted(acc.items(), key=key)[:top]:
        wi = a["Instructions Executed"] or 1
        wf = a["L1 Wavefronts Shared"]
        ideal = a["L1 Wavefronts Shared Ideal"]
        conf = f"{wf / ideal:5.2f}" if ideal else "    -"
        print(f"{a['Instructions Executed'] / tot:5.3f}  {a['Warp Stall Sampling (All Samples)'] / ts:5.3f}  "
              f"{a['Thread Instructions Executed'] / wi:7.1f}  {conf:>13}  {k[0]}:{k[1]}  {src.get(k, '')}")
    if "--opcodes" in sys.argv:
        print("# opcode mix")
        for o, v in ops.most_common(25):
            print(f"{v / tot:6.3f} {o}")


if __name__ == "__main__":
    main()
