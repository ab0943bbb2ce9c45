"""Per-instruction view of an ncu --set full capture (needs --import-source):
hot basic blocks by executed instructions, with stall samples.

    ncu -i prof.ncu-rep --page source --csv --print-source sass > x.csv
    python tools/sass_profile.py x.csv [top_blocks]
"""
import csv
import re
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    ins = []
    for r in rows[2:]:
        try:
            ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
        except (ValueError, IndexError):
            pass
    tot_ex = sum(x[2] for x in ins)
    tot_st = sum(x[3] for x in ins)
    # stall-reason columns
    reasons = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
    print(f"instructions executed (warp-level): {tot_ex:.4g}; stall samples {tot_st}")
    # group consecutive instructions with equal execution count into blocks
    blocks, cur = [], []
    for x in ins:
        if cur and x[2] != cur[-1][2]:
            blocks.append(cur)
            cur = []
        cur.append(x)
    if cur:
        blocks.append(cur)
    blocks.sort(key=lambda b: -sum(x[2] for x in b))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    for b in blocks[:top]:
        ex = sum(x[2] for x in b)
        st = sum(x[3] for x in b)
        ops = {}
        for x in b:
            op = re.sub(r"^@!?U?P\w+\s+", "", x[1]).split(" ")[0]
            ops[op] = ops.get(op, 0) + 1
        print(f"-- block @{b[0][0]:#x}: {len(b)} instr x {b[0][2]} = {100*ex/tot_ex:.1f}% of "
              f"executed, {100*st/max(tot_st,1):.1f}% of stall samples")
        print("   " + ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda t: -t[1])))


if __name__ == "__main__":
    main()
