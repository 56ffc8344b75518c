"""Classify the SASS of a kernel's main loop by pipe (rough Blackwell mapping)."""
import re, subprocess, sys, collections
binf, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", binf], capture_output=True, text=True).stdout
blocks = out.split("Function : ")
body = [b for b in blocks if b.startswith(fn)]
if not body:
    print("not found"); sys.exit(1)
lines = [l for l in body[0].split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", l)
    if not m: continue
    addr = int(m.group(1), 16); txt = m.group(2).strip()
    txt = re.sub(r"^@!?U?P[T0-9]+\s+", "", txt)
    ins.append((addr, txt))
# find the largest backward-branch loop
loops = []
for addr, txt in ins:
    m = re.match(r"BRA\s+(?:`?\(?\.?L?_?x?_?\d*\)?)?\s*0x([0-9a-f]+)", txt)
    if txt.startswith("BRA") and not txt.startswith("BRA.U"):
        mm = re.search(r"0x([0-9a-f]+)", txt)
        if mm and int(mm.group(1), 16) < addr:
            loops.append((addr - int(mm.group(1), 16), int(mm.group(1), 16), addr))
loops.sort(reverse=True)
if len(sys.argv) > 3:  # the largest loop containing this opcode
    loops = [l for l in loops if any(l[1] <= a <= l[2] and t.startswith(sys.argv[3]) for a, t in ins)]
_, lo, hi = loops[0]
body_ins = [t for a, t in ins if lo <= a <= hi]
pipe = collections.Counter(); ops = collections.Counter()
def cls(op):
    if op.startswith(("IMAD", "IMUL")): return "fmaheavy"
    if op.startswith(("FFMA", "FADD", "FMUL")): return "fma"
    if op.startswith(("DMUL", "DADD", "DFMA", "DSETP")): return "fp64"
    if op.startswith(("I2F", "F2F", "F2I", "MUFU")): return "xu/conv"
    if op.startswith(("LDG", "STG", "LDS", "STS", "LDC", "SHFL")): return "mio"
    if op.startswith(("U", "LDCU", "S2UR")): return "uniform"
    if op.startswith(("BRA", "EXIT", "NOP")): return "ctrl"
    if op.startswith("VIADD"): return "viadd"
    return "alu"
for t in body_ins:
    op = t.split()[0]
    ops[op] += 1; pipe[cls(op)] += 1
print(f"loop {lo:#x}-{hi:#x}: {len(body_ins)} instrs")
print(dict(pipe)); print(dict(ops.most_common()))
