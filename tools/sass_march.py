"""SASS instructions per march step of env_step_kernel<kSmem=1, kRec=0> (host-side tool).

    python tools/sass_march.py [lib.so ...]

Disassembles each library with line info, takes the instructions whose
innermost source line lies inside ray_step() (csrc/sp_env.cu), and divides by
the inlined copies (2 rays x SP_MARCH_GROUP steps x 2 ray phases).  Also lists
the opcode mix of one copy's worth.
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2305_04180_b200", "csrc", "sp_env.cu")
KERNEL = "_ZN2sp15env_step_kernelILb1ELb0EEEvNS_6EnvDevENS_8StepArgsE"


def step_lines():
    lines = open(SRC).read().split("\n")
    start = next(i for i, l in enumerate(lines) if "bool ray_step(" in l) + 1
    end = next(i for i in range(start, len(lines)) if lines[i].startswith("}")) + 1
    return start, end


def main(libs):
    lo, hi = step_lines()
    for lib in libs or [os.path.join(ROOT, "paper_2305_04180_b200", "_lib", "libsparrow.so")]:
        with tempfile.TemporaryDirectory() as td:
            subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=td,
                           capture_output=True, check=True)
            cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
            txt = subprocess.run(["nvdisasm", "-gi", os.path.join(td, cub)], capture_output=True,
                                 text=True).stdout
        a = txt.index(".text." + KERNEL + ":")
        b = txt.find("\n.text.", a + 10)
        body = txt[a:b if b > 0 else None].split("\n")
        cur, ops = None, collections.Counter()
        n, fresh = 0, True
        for l in body:
            if l.strip().startswith("//##"):  # innermost first, then the inlining chain
                if fresh:
                    m = re.search(r'sp_env\.cu", line (\d+)', l)
                    cur = int(m.group(1)) if m and "sp_env.cu\", line" in l.split("inlined")[0] else None
                    fresh = False
                continue
            fresh = True
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
            if m and cur is not None and lo <= cur <= hi:
                n += 1
                ops[m.group(2).split(".")[0]] += 1
        copies = 2 * 4 * 2
        print(f"{os.path.basename(lib)}: {n} instructions in ray_step copies -> {n / copies:.1f} per step")
        print("   ", " ".join(f"{k}:{v / copies:.2g}" for k, v in ops.most_common()))


if __name__ == "__main__":
    main(sys.argv[1:])
