"""List the innermost loops of a kernel's SASS with their instruction mix (runs here, no GPU).

    python tools/sass_loops.py <object.o|lib.so> <kernel-name-regex>

For each backward branch: address range, instruction count, FP64 (DFMA/DMUL/DADD), MUFU,
UMOV/IMAD.MOV (re-materialised constants), loads — to compare A/B builds before spending GPU time.
"""

import re
import subprocess
import sys


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not re.search(pat, name):
            continue
        ins = []
        for line in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        addr = {a: k for k, (a, _) in enumerate(ins)}
        print(name[:110])
        for k, (a, t) in enumerate(ins):
            m = re.search(r"BRA (0x[0-9a-f]+)", t)
            if not m or int(m.group(1), 16) >= a:
                continue
            s = addr.get(int(m.group(1), 16))
            if s is None:
                continue
            body = [x for _, x in ins[s:k + 1]]
            ops = [re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] for x in body]
            fp64 = sum(o.split(".")[0] in ("DFMA", "DMUL", "DADD") for o in ops)
            cnt = lambda p: sum(o.startswith(p) for o in ops)
            print(f"  loop {ins[s][0]:#07x}-{a:#07x}: {len(body):4d} instr, fp64 {fp64:3d}, mufu {cnt('MUFU'):2d}, "
                  f"umov {cnt('UMOV'):2d}, imad.mov {cnt('IMAD.MOV'):2d}, ldg {cnt('LDG'):2d}, lds {cnt('LDS'):2d}, "
                  f"shfl {cnt('SHFL'):2d}")


if __name__ == "__main__":
    main()
