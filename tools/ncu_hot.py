"""Aggregate ncu SASS source-page stall samples by instruction class and by
code region (between BAR.SYNC barriers)."""
import csv, subprocess, sys, collections, re

def main(path, kid=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    # split per kernel (each block starts with "Kernel Name")
    blocks, cur = [], []
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            if cur: blocks.append(cur)
            cur = [ln]
        else:
            cur.append(ln)
    if cur: blocks.append(cur)
    b = blocks[kid]
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    si, ni, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    byop = collections.Counter(); region = collections.Counter(); execd = collections.Counter()
    reg = 0
    for r in rows[1:]:
        src = r[si].strip(); s = int(r[ni] or 0); e = int(r[ei] or 0)
        op = re.sub(r"^@!?U?P\d+\s+", "", src).split(" ")[0]
        byop[op] += s; execd[op] += e
        region[reg] += s
        if "BAR.SYNC" in src: reg += 1
    tot = sum(byop.values())
    print("total samples", tot)
    for op, s in byop.most_common(15):
        print(f"{op:14s} {100*s/tot:5.1f}%  executed {execd[op]}")
    print("regions (split at BAR.SYNC):", {k: round(100*v/tot,1) for k,v in region.items()})

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
