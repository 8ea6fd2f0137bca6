"""Per-region (between BAR.SYNCs) stall breakdown and instruction mix from the
ncu SASS source page."""
import csv, subprocess, sys, collections, re

def main(path, kid=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], []
    for ln in out.splitlines():
        if ln.startswith('"Kernel Name"'):
            if cur: blocks.append(cur)
            cur = [ln]
        else:
            cur.append(ln)
    blocks.append(cur)
    rows = list(csv.reader(blocks[kid][1:]))
    hdr = rows[0]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    reg = 0
    R = collections.defaultdict(collections.Counter)
    E = collections.defaultdict(collections.Counter)
    for r in rows[1:]:
        src = r[si].strip()
        op = re.sub(r"^@!?U?P\d+\s+", "", src).split(" ")[0]
        for h in stall_cols:
            R[reg][h] += int(r[hdr.index(h)] or 0)
        E[reg][op] += int(r[ei] or 0)
        if "BAR.SYNC" in src:
            reg += 1
    tot = sum(sum(c.values()) for c in R.values())
    for k in sorted(R):
        s = sum(R[k].values())
        top = ", ".join(f"{h[6:]} {100*v/s:.0f}%" for h, v in R[k].most_common(6))
        ins = sum(E[k].values())
        fp = E[k]["DFMA"] + E[k]["DADD"] + E[k]["DMUL"]
        print(f"region {k}: {100*s/tot:.1f}% of samples; instr {ins/1e6:.1f}M, FP64 {fp/1e6:.1f}M ({100*fp/max(ins,1):.0f}%) | {top}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
