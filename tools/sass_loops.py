"""Static view of a kernel's SASS: loops (backward branches), their opcode mix
and the sum of the compiler-encoded stall counts (the minimum cycles one warp
needs per trip when nothing else stalls it).

    python tools/sass_loops.py LIB.so MANGLED_KERNEL_NAME [--mix LO HI]

Control bits (Volta+ 128-bit encoding): high word bits 41-44 = stall count.
"""
import collections
import re
import subprocess
import sys

FP64 = ("DFMA", "DMUL", "DADD", "DSETP", "MUFU")


def decode(lib, fun):
    txt = subprocess.run(["cuobjdump", "-sass", "-fun", fun, lib], capture_output=True,
                         text=True).stdout.split("\n")
    pat = re.compile(r"^\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);\s+/\* (0x[0-9a-f]{16}) \*/")
    pat2 = re.compile(r"^\s+/\* (0x[0-9a-f]{16}) \*/")
    ins, i = [], 0
    while i < len(txt):
        m = pat.match(txt[i])
        if m and i + 1 < len(txt):
            m2 = pat2.match(txt[i + 1])
            if m2:
                hi = int(m2.group(1), 16)
                ins.append((int(m.group(1), 16), m.group(2).strip(), (hi >> 41) & 0xF))
                i += 2
                continue
        i += 1
    return ins


def opcode(t):
    tt = t.split()
    op = tt[1] if tt[0].startswith("@") else tt[0]
    return op.split(".")[0]


def main():
    lib, fun = sys.argv[1], sys.argv[2]
    ins = decode(lib, fun)
    if not ins:
        sys.exit("kernel not found (name must be the mangled one)")
    addr = {a: i for i, (a, *_) in enumerate(ins)}
    print(f"{len(ins)} instructions")
    for i, (a, t, s) in enumerate(ins):
        if "BRA" in t:
            m = re.search(r"0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
                body = ins[addr[int(m.group(1), 16)]:i + 1]
                nfp = sum(1 for x in body if opcode(x[1]) in FP64)
                nbr = sum(1 for x in body if opcode(x[1]) in ("BRA", "BSSY", "BSYNC"))
                print(f"loop {int(m.group(1), 16):#x}..{a:#x}: {len(body)} instr, {nfp} FP64, "
                      f"{nbr} control, stall sum {sum(x[2] for x in body)}")
    if "--mix" in sys.argv:
        k = sys.argv.index("--mix")
        lo, hi = int(sys.argv[k + 1], 16), int(sys.argv[k + 2], 16)
        c, st = collections.Counter(), collections.Counter()
        for a, t, s in ins:
            if lo <= a <= hi:
                c[opcode(t)] += 1
                st[opcode(t)] += s
        for op, n in c.most_common():
            print(f"  {op:10s} {n:5d}  stall {st[op]}")


if __name__ == "__main__":
    main()
