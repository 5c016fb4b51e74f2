"""Size of the march loop in SASS: the smallest backward-branch range of a
kernel that contains `need` table loads (LDS.S8 / LDS.U8).  Usage:
python tools/debug/sass_loop.py [lib.so] [kernel-substring] [need]"""
import re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2305_04180_b200/_lib/libsparrow.so"
kern = sys.argv[2] if len(sys.argv) > 2 else "env_step_kernelILb1E"
need = int(sys.argv[3]) if len(sys.argv) > 3 else 4
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
body, cur = [], None
for l in out.split("\n"):
    m = re.match(r"\s+Function : (\S+)", l)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and cur and kern in cur:
        body.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for i, (addr, ins) in enumerate(body):
    m = re.search(r"BRA\s+(?:\S+\s+)?0x([0-9a-f]+)", ins)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= addr:
        continue
    seg = [x for a, x in body if tgt <= a <= addr]
    loads = sum(1 for x in seg if re.search(r"LDS\.[SU]8", x))
    if loads >= need and (best is None or len(seg) < len(best[2])):
        best = (tgt, addr, seg)
if best is None:
    sys.exit("no loop found")
tgt, addr, seg = best
ops = {}
for x in seg:
    op = re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0]
    ops[op] = ops.get(op, 0) + 1
print(f"{kern}: loop 0x{tgt:x}..0x{addr:x}: {len(seg)} instructions, "
      f"{sum(1 for x in seg if re.search(r'LDS[.][SU]8', x))} table loads")
print(" ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])))
if "-v" in sys.argv:
    print("\n".join(seg))
