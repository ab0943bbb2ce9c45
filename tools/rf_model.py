"""Static register-file read model of a kernel's hottest basic block.

B200 microbenchmarks (tools/microbench/rfbench.cu, profiles/r02_rfbench.txt)
fit ~0.56 scheduler cycles per 32-bit vector-register operand read: FFMA2
P-S-P (5 reads) 2.75 cycles, FMUL2 P-P (4) 2.2, + LEA.HI (2 reads) +1.3,
+ IMNMX (2) +1.05.  This counts, per instruction, the vector registers it
reads (a .F32x2 pair = 2, RZ/UR/immediates/constants free), minus operands
marked .reuse on the previous instruction in the same slot, and reports
reads, issue slots and FMA-pipe cycles of the block.

usage: python tools/rf_model.py build/obj/crossing.o cross_filter_kernelILb0E [OPCODE]
"""
import re
import subprocess
import sys

PIPE2 = ("FFMA2", "FMUL2", "FADD2")


def hot_block(obj, pat, key):
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
    best = max(sum(key in t for t in b) for b in blocks)
    hot = [b for b in blocks if sum(key in t for t in b) == best]
    return hot if ALL else hot[0]


ALL = False


def operands(txt):
    txt = re.sub(r"^@!?U?P\w+\s+", "", txt)
    parts = txt.split(None, 1)
    op = parts[0]
    args = [a.strip() for a in parts[1].split(",")] if len(parts) > 1 else []
    return op, args


def reads(op, args):
    """[(slot, reg, width, reuse)] of the vector registers an instruction reads."""
    out = []
    srcs = args[1:] if not op.startswith(("ST", "BRA", "ISETP", "FSETP", "DSETP", "VOTE")) else args
    if op.startswith(("ISETP", "FSETP", "DSETP")):
        srcs = args[2:]
    slot = 0
    for a in srcs:
        m = re.match(r"-?\|?(R\d+)(\.reuse)?(\.F32x2[.\w]*)?", a.replace("[", "").replace("]", ""))
        if m and m.group(1) != "RZ":
            width = 2 if m.group(3) or op.startswith("D") or ".64" in op else 1
            out.append((slot, m.group(1), width, bool(m.group(2))))
        slot += 1
    return out


def block_reads(blk):
    total = 0
    cache = {}
    for txt in blk:
        op, args = operands(txt)
        nc = {}
        for slot, reg, w, reuse in reads(op, args):
            if cache.get(slot) != reg:
                total += w
            if reuse:
                nc[slot] = reg
        cache = nc
    return total


def main():
    global ALL
    obj, pat = sys.argv[1], sys.argv[2]
    key = sys.argv[3] if len(sys.argv) > 3 else "FFMA2"
    ALL = True
    for blk in hot_block(obj, pat, key):
        report(blk)


def report(blk):
    total = pipe = 0
    cache = {}
    for txt in blk:
        op, args = operands(txt)
        r = 0
        newcache = {}
        for slot, reg, w, reuse in reads(op, args):
            if cache.get(slot) != reg:
                r += w
            if reuse:
                newcache[slot] = reg
        cache = newcache
        total += r
        if op in PIPE2:
            pipe += 2
        elif op in ("FFMA", "FMUL", "FADD"):
            pipe += 1
    n = len(blk)
    print(f"block: {n} instructions, {total} vector-register reads (x0.56 = {0.56 * total:.1f} "
          f"cycles), FMA-pipe {pipe} cycles, issue {n} cycles")


if __name__ == "__main__":
    main()


def bank_cycles(blk, nbanks=2):
    """Alternative model: an instruction costs max over register banks of its
    fresh (non-reused) 32-bit reads, register Rn in bank n % nbanks (a pair
    touches two banks); pipes and issue cost at least 1 (FFMA2 class 2)."""
    cache = {}
    total = 0
    for txt in blk:
        op, args = operands(txt)
        banks = [0] * nbanks
        nc = {}
        for slot, reg, w, reuse in reads(op, args):
            if cache.get(slot) != reg:
                r = int(reg[1:])
                for k in range(w):
                    banks[(r + k) % nbanks] += 1
            if reuse:
                nc[slot] = reg
        cache = nc
        floor = 2 if op in PIPE2 else 1
        total += max(max(banks), floor)
    return total
