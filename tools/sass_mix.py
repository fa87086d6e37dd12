"""Opcode mix of the SASS of one kernel (whole function and its hottest loop).

usage: python tools/sass_mix.py <lib.so> <function-substring> [more substrings...]
The "loop" section counts the instructions between the target of the largest
backward branch and the branch itself -- the per-block body of the hash
kernels.  Used to check that rotates/booleans/adds map onto SHF/LEA.HI/LOP3/
IADD3 and to estimate ALU-vs-FMA pipe pressure before spending GPU time.
"""
import collections
import re
import subprocess
import sys

ALU = {"LOP3", "SHF", "IADD3", "PRMT", "LEA", "ISETP", "SEL", "PLOP3", "IMNMX", "VIMNMX", "SHL", "SHR", "FLO", "POPC"}
FMA = {"IMAD", "IMUL", "FFMA", "VIADD", "IADD"}  # VIADD: Blackwell integer add issued on the FMA-side datapath


def functions(sass):
    cur, buf = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, buf
            cur, buf = m.group(1), []
        elif cur:
            buf.append(line)
    if cur:
        yield cur, buf


def parse(lines):
    ins = []
    for line in lines:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?\s*([^;]*);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), (m.group(4) or ""), m.group(5)))
    return ins


def mix(ins):
    c = collections.Counter(op for _, op, _, _ in ins)
    alu = sum(v for k, v in c.items() if k in ALU)
    fma = sum(v for k, v in c.items() if k in FMA)
    return c, alu, fma


def main():
    lib, pats = sys.argv[1], sys.argv[2:]
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    for name, lines in functions(sass):
        if not all(p in name for p in pats):
            continue
        ins = parse(lines)
        c, alu, fma = mix(ins)
        print(f"== {name}: {len(ins)} instructions  alu-pipe~{alu} fma-pipe~{fma}")
        # largest backward branch = main loop
        best = None
        for addr, op, mod, args in ins:
            if op == "BRA":
                m = re.search(r"0x([0-9a-f]+)", args)
                if m and int(m.group(1), 16) < addr:
                    span = addr - int(m.group(1), 16)
                    if not best or span > best[0]:
                        best = (span, int(m.group(1), 16), addr)
        if best:
            body = [x for x in ins if best[1] <= x[0] <= best[2]]
            bc, balu, bfma = mix(body)
            print(f"   loop [{best[1]:#x},{best[2]:#x}] {len(body)} instr  alu~{balu} fma~{bfma}")
            print("   ", ", ".join(f"{k}:{v}" for k, v in bc.most_common(18)))


if __name__ == "__main__":
    main()
