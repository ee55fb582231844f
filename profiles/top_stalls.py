"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys


def top(rep, n=25, kernel_idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    s = starts[kernel_idx]
    e = starts[kernel_idx + 1] - 1 if kernel_idx + 1 < len(starts) else len(rows)
    h = rows[s]
    body = [r for r in rows[s + 1:e] if len(r) == len(h)]
    si, ni = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(int(r[si]) for r in body)
    body.sort(key=lambda r: -int(r[si]))
    lines = [f"total samples {tot}, {len(body)} SASS lines"]
    for r in body[:n]:
        lines.append(f"{int(r[si]) / tot:6.3f}  {r[0][-5:]}  {r[ni].strip()[:90]}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(top(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, int(sys.argv[3]) if len(sys.argv) > 3 else 0))
