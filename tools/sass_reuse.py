"""Operand-reuse audit of a kernel's hot loop (SASS of an object or .so).

For the innermost loop with the most FFMA2 (or DFMA) instructions: how many of
its three-distinct-operand accumulates (acc = d*w + acc) carry a `.reuse` flag --
ptxas keeps w in the operand reuse cache for the next instruction only when it
schedules the x/y/z accumulates of a weight next to each other (two of every
triple can reuse at best) -- and the same for the FADD2 source operand.
usage: python tools/sass_reuse.py LIB KERNEL_SUBSTRING [--f64]
e.g.   python tools/sass_reuse.py paper_2203_08263_b200/libnbody_b200.so \\
           step_kernelINS_8CoreF32MILb0ELb0EEELi256ELi256ELi1ELi16ELb0ELb0
(profiles/r02/variants_r02_split_acc.txt)"""
import re
import subprocess
import sys

BRA = re.compile(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)")


def main():
    lib, pat = sys.argv[1], sys.argv[2]
    f64 = "--f64" in sys.argv
    op = "DFMA" if f64 else "FFMA2"
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s+Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        if pat not in name:
            continue
        ins = []
        for line in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), re.sub(r"^@!?U?P\d+\s+", "", m.group(2).strip())))
        best = None
        for a, t in ins:
            m = BRA.search(t)
            if not (m and int(m.group(1), 16) < a):
                continue
            lo = int(m.group(1), 16)
            body = [x for x in ins if lo <= x[0] <= a]
            back = sum(1 for x in body if BRA.search(x[1]) and int(BRA.search(x[1]).group(1), 16) < x[0])
            n = sum(1 for x in body if x[1].startswith(op))
            if back == 1 and (best is None or n > best[0]):
                best = (n, lo, a, body)
        if best is None:
            print(name[:80], "no loop")
            continue
        n, lo, hi, body = best
        acc = acc_reuse = add = add_reuse = 0
        for _, t in body:
            m = re.match(rf"{op} (R\d+), (-?R\d+)(\S*), (-?R\d+)(\S*), (-?R\d+)", t)
            if m and len({m.group(2).strip("-"), m.group(4).strip("-"), m.group(6).strip("-")}) == 3 and \
                    (f64 or ("x2" in m.group(3) and "x2" in m.group(5))):
                acc += 1
                acc_reuse += "reuse" in t
            if t.startswith("FADD2"):
                add += 1
                add_reuse += "reuse" in t
        print(f"{name[:80]}\n  loop {lo:#x}-{hi:#x}: {len(body)} instructions, {n} {op}; three-operand accumulates {acc}, "
              f"with .reuse {acc_reuse} (max {acc * 2 // 3})" + ("" if f64 else f"; FADD2 {add}, with .reuse {add_reuse}"))


if __name__ == "__main__":
    main()
