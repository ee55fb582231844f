"""Instruction mix of one kernel from an ncu report (source page, SASS):
warp-level instructions executed, shared wavefronts and stall samples per
opcode."""
import collections
import csv
import subprocess
import sys


def mix(rep, kernel_idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    s = starts[kernel_idx]
    e = starts[kernel_idx + 1] - 1 if kernel_idx + 1 < len(starts) else len(rows)
    h = rows[s]
    body = [r for r in rows[s + 1:e] if len(r) == len(h)]
    ie, ws, st = h.index("Instructions Executed"), h.index("L1 Wavefronts Shared"), h.index("Warp Stall Sampling (All Samples)")
    tg = h.index("L1 Tag Requests Global")
    agg = collections.defaultdict(lambda: [0, 0, 0, 0])
    for r in body:
        ins = r[1].strip().split()
        op = ins[1] if ins and ins[0].startswith("@") and len(ins) > 1 else (ins[0] if ins else "?")
        a = agg[op]
        a[0] += int(r[ie] or 0); a[1] += int(r[ws] or 0); a[2] += int(r[st] or 0); a[3] += int(r[tg] or 0)
    tot = sum(a[0] for a in agg.values())
    print(f"{'opcode':24s} {'inst':>12s} {'frac':>6s} {'shared_wf':>10s} {'l1_tag_glb':>10s} {'stall':>7s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
        print(f"{k:24s} {a[0]:12d} {a[0] / tot:6.3f} {a[1]:10d} {a[3]:10d} {a[2]:7d}")
    print("total inst", tot)


if __name__ == "__main__":
    mix(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
