"""Instruction mix of the hottest basic block of a kernel's SASS.

usage: python tools/sass_loop.py build/obj/crossing.o cross_filter_kernelILb1E [OPCODE]

Splits the function into basic blocks at branch targets and branches, picks
the block with the most instructions of OPCODE (default FFMA2) and prints its
length and opcode histogram -- a static check of instructions per pair before
spending GPU time.
"""
import collections
import re
import subprocess
import sys


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    key = sys.argv[3] if len(sys.argv) > 3 else "FFMA2"
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True,
                          check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    body = next(f for f in funcs[1:] if pat in f.split("\n", 1)[0])
    ins = []
    for line in body.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    targets = set()
    for _, txt in ins:
        m = re.search(r"BRA(?:\.\w+)*\s+(?:\S+,\s*)?(?:`\()?0x([0-9a-f]+)", txt)
        if m:
            targets.add(int(m.group(1), 16))
    blocks, cur = [], []
    for addr, txt in ins:
        if addr in targets and cur:
            blocks.append(cur)
            cur = []
        cur.append(txt)
        if re.search(r"\bBRA\b|EXIT|RET", txt):
            blocks.append(cur)
            cur = []
    if cur:
        blocks.append(cur)

    def op(t):
        t = re.sub(r"^@!?U?P\w+\s+", "", t)
        return t.split()[0]

    top = max(sum(op(t) == key for t in b) for b in blocks)
    for best in blocks:  # every block with the top count (e.g. diagonal + off-diagonal)
        hist = collections.Counter(op(t) for t in best)
        if hist[key] != top:
            continue
        print(f"block: {len(best)} instructions, {hist[key]} {key}")
        for o, c in hist.most_common():
            print(f"  {c:5d} {o}")


if __name__ == "__main__":
    main()
