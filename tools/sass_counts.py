"""Per-kernel SASS instruction counts of libpgx.so (static, no GPU needed).

Runs `cuobjdump -sass` on the built library, demangles each function name and counts the
mnemonics that show whether a kernel does what DESIGN.md §4 says it does: 128-bit global
loads/stores (LDG/STG .128), TMA bulk copies (UBLKCP / UTMALDG / UTMASTG), mbarrier ops
(SYNCS), system-scope fences (MEMBAR.ALL.SYS / FENCE), strong system loads/stores (the flag
protocol), multimem (NVLS) and warp votes.  Output: one JSON object per kernel instance
(static counts, i.e. instructions in the binary, not executed counts).

  python tools/sass_counts.py [--lib paper_1706_00095_b200/libpgx.so] [--match k_twoshot]
"""

from __future__ import annotations

import argparse
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PATTERNS = {  # matched against the opcode (first token after the address, predicate stripped)
    "LDG.128": r"^LDG\.\S*128",
    "STG.128": r"^STG\.\S*128",
    "LDG": r"^LDG\.",
    "STG": r"^STG\.",
    "LD.STRONG.SYS": r"^LDG\.\S*STRONG\.SYS",
    "ST.STRONG.SYS": r"^STG\.\S*STRONG\.SYS",
    "RED/ATOM.SYS": r"^(?:REDG|ATOMG)\.\S*SYS",
    "MEMBAR.SYS": r"^MEMBAR\.\S*SYS",
    "MEMBAR.GPU": r"^MEMBAR\.\S*GPU",
    "FENCE.VIEW.ASYNC": r"^FENCE\.VIEW\.ASYNC",
    "UBLKCP": r"^UBLKCP",
    "UTMALDG": r"^UTMALDG",
    "UTMASTG": r"^UTMASTG",
    "SYNCS": r"^SYNCS\.",
    "MULTIMEM": r"^(?:LDG|STG|REDG|ATOMG)MC",
    "VOTE": r"^VOTE",
    "BAR.SYNC": r"^BAR\.SYNC",
    "NANOSLEEP": r"^NANOSLEEP",
    "DFMA": r"^DFMA",
    "FFMA": r"^FFMA",
}


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
    return out.splitlines()


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = re.sub(r"pgx::", "", name)
    return re.sub(r"\(.*\)$", "", name)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_1706_00095_b200", "libpgx.so"))
    ap.add_argument("--match", default="")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    mangled = [f.split("\n", 1)[0].strip() for f in funcs]
    names = demangle(mangled)
    rx = {k: re.compile(v) for k, v in PATTERNS.items()}
    for name, body in zip(names, funcs):
        name = short(name)
        if a.match and a.match not in name:
            continue
        ops = [m.group(1) for m in re.finditer(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_.]*)", body)]
        counts = {"instructions": len(ops)}
        for k, r in rx.items():
            n = sum(1 for op in ops if r.search(op))
            if n:
                counts[k] = n
        print(json.dumps({"kernel": name, **counts}))


if __name__ == "__main__":
    main()
