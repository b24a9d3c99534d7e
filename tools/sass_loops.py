"""List the innermost loops of a kernel's SASS with their instruction mix (runs here, no GPU).

    python tools/sass_loops.py <object.o|lib.so> <kernel-name-regex>

For each backward branch: address range, instruction count, FP64 (DFMA/DMUL/DADD), MUFU,
UMOV/IMAD.MOV (re-materialised constants), loads — to compare A/B builds before spending GPU time.
`fp64_per_pair()` is what bench.py reports as the implemented FP64-pipe work per ordered pair.
"""

import re
import subprocess
import sys


def loops(obj: str, pat: str) -> list:
    """[{kernel, start, end, instr, fp64, mufu, umov, imad_mov, ldg, lds, shfl}] of every loop."""
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    res = []
    for f in re.split(r"\n\s+Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        if not re.search(pat, name):
            continue
        ins = []
        for line in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        addr = {a: k for k, (a, _) in enumerate(ins)}
        for k, (a, t) in enumerate(ins):
            # BRA 0x.., @P0 BRA 0x.., BRA.U UP0, 0x.. (uniform-predicate back edges of unrolled loops)
            m = re.search(r"BRA\S*\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", t)
            if not m or int(m.group(1), 16) >= a:
                continue
            s = addr.get(int(m.group(1), 16))
            if s is None:
                continue
            body = [x for _, x in ins[s:k + 1]]
            ops = [re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] for x in body]
            cnt = lambda p: sum(o.startswith(p) for o in ops)  # noqa: E731
            res.append(dict(kernel=name, start=ins[s][0], end=a, instr=len(body), fp64_reads=_fp64_reads(body),
                            fp64=sum(o.split(".")[0] in ("DFMA", "DMUL", "DADD") for o in ops),
                            mufu=cnt("MUFU"), umov=cnt("UMOV"), imad_mov=cnt("IMAD.MOV"), ldg=cnt("LDG"),
                            lds=cnt("LDS"), shfl=cnt("SHFL")))
    return res


# FP64-pipe issue cycles of an instruction by its fresh 64-bit register operands (not from the
# reuse cache, a uniform register, the constant bank or an immediate), measured on a B200 by
# tools/issue_probe2.cu: two operands sustain the pipe's 2 cycles per warp instruction, three
# take ~3.2 (0.311 instead of 0.478 instructions per clock per sub-partition).
FP64_ISSUE_CYCLES = {0: 2.0, 1: 2.0, 2: 2.0, 3: 3.2}


def _fp64_reads(body) -> dict:
    """{fresh 64-bit register source operands: count} over the FP64 instructions of a loop body."""
    hist = {}
    for x in body:
        m = re.match(r"(?:@!?U?P\w+\s+)?(\S+)\s*(.*)", x)
        if not m or m.group(1).split(".")[0] not in ("DFMA", "DMUL", "DADD"):
            continue
        srcs = [a.strip().lstrip("-|").rstrip("|") for a in m.group(2).split(",")][1:]
        n = len({a for a in srcs if re.match(r"R\d+", a) and ".reuse" not in a})  # distinct registers
        hist[n] = hist.get(n, 0) + 1
    return hist


def operand_read_ceiling(loop: dict) -> float:
    """Upper bound of the FP64-pipe utilisation of a loop's instruction mix: 2 cycles per FP64
    instruction over the cycles its operand reads hold the pipe's issue (FP64_ISSUE_CYCLES)."""
    h = loop["fp64_reads"]
    n = sum(h.values())
    return 2.0 * n / sum(FP64_ISSUE_CYCLES.get(k, 3.2) * v for k, v in h.items()) if n else 0.0


def fp64_per_pair(obj: str, pat: str, symmetric: bool):
    """FP64-pipe instructions per ORDERED pair in the hottest loop of the kernel: the loop with the
    most FP64 instructions; every conical pair evaluation issues one MUFU.RSQ64H, so the loop's
    pair count is its MUFU count (an unordered pair feeds two ordered pairs in the symmetric
    kernel).  Returns (fp64 per ordered pair, loop dict) or (None, None)."""
    ls = [x for x in loops(obj, pat) if x["mufu"] > 0]
    # innermost pair loops only: a loop around another loop with MUFU (phase / tile loops) mixes in
    # the diagonal one-sided tiles and the setup code
    ls = [x for x in ls if not any(y is not x and y["kernel"] == x["kernel"] and x["start"] <= y["start"]
                                   and y["end"] <= x["end"] for y in ls)]
    if not ls:
        return None, None
    best = max(ls, key=lambda x: x["fp64"])
    return best["fp64"] / (best["mufu"] * (2 if symmetric else 1)), best


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    last = None
    for x in loops(obj, pat):
        if x["kernel"] != last:
            print(x["kernel"][:110])
            last = x["kernel"]
        print(f"  loop {x['start']:#07x}-{x['end']:#07x}: {x['instr']:4d} instr, fp64 {x['fp64']:3d}, "
              f"mufu {x['mufu']:2d}, umov {x['umov']:2d}, imad.mov {x['imad_mov']:2d}, ldg {x['ldg']:2d}, "
              f"lds {x['lds']:2d}, shfl {x['shfl']:2d}, fp64 by fresh register operands {dict(sorted(x['fp64_reads'].items()))}"
              f" -> operand-read ceiling {operand_read_ceiling(x):.2f}")


if __name__ == "__main__":
    main()
