"""Per-kernel SASS instruction summary of the in-tree library (cuobjdump -sass).

    python scripts/sass_summary.py > profiles/round2_sass.md

For each kernel: instruction count and the mnemonics that show how it moves
memory on sm_100a -- 128-bit global loads/stores (LDG.E.128 / STG.E.128 with
their cache qualifiers), bulk copies and mbarriers (UBLKCP, SYNCS), shuffles,
atomics and fences.  No tensor-core (UTC*MMA) or TMEM (LDTM/STTM) instruction
is expected: nothing on this path is a contraction.
"""
from __future__ import annotations

import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2104_06069_b200", "libbitlamb_b200.so")
KEYS = ["LDG", "STG", "LDS", "STS", "SHFL", "UBLKCP", "SYNCS", "ATOM", "ATOMG", "RED", "MEMBAR", "FENCE",
        "DADD", "FADD", "FMUL", "MUFU", "BAR", "UTCHMMA", "UTCQMMA", "LDTM", "STTM"]


def main() -> None:
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kern, per = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            kern = re.sub(r"bl::\(anonymous namespace\)::", "", kern).split("(")[0]
            per[kern] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m and kern:
            full = m.group(1)
            per[kern]["_total"] += 1
            base = full.split(".")[0]
            if base in ("LDG", "STG") and ".128" in full:
                per[kern][full] += 1
            per[kern][base] += 1
    print("# SASS summary of libbitlamb_b200.so (sm_100a)\n")
    print("`cuobjdump -sass paper_2104_06069_b200/libbitlamb_b200.so`, counted per kernel by "
          "`scripts/sass_summary.py`. Static instruction counts (not executed counts).\n")
    keep = [k for k in per if re.search(r"k1_|k3_|k5_|k6_|kw1|kw2|k_small|k_lossless|k_step_gate|k_check_finite", k)]
    for k in keep:
        c = per[k]
        wide = ", ".join(f"{n} {v}" for n, v in sorted(c.items()) if n.startswith(("LDG.", "STG.")))
        other = ", ".join(f"{n} {c[n]}" for n in KEYS if c.get(n))
        print(f"## {k}\n\n- instructions: {c['_total']}\n- 128-bit global: {wide or 'none'}\n- {other}\n")


if __name__ == "__main__":
    main()
