"""Per-kernel SASS instruction summary of libocean_b200.so (cuobjdump, no GPU
needed): total instructions and the counts of the mnemonics that prove the
Blackwell data paths (TMA: UTMALDG / UTMASTG / UBLKCP; mbarrier: SYNCS), the
shared-memory exchange (LDS / STS), global traffic (LDG / STG) and FP32 / FP64
arithmetic (scalar and packed fp32x2), written to profiles/sass_summary_<tag>.txt.

    python tools/sass_summary.py r02
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2503_03326_b200", "lib", "libocean_b200.so")
KEYS = ["UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG", "BAR", "SHFL",
        "FFMA", "FADD", "FMUL", "FFMA2", "FADD2", "FMUL2", "DFMA", "DADD", "DMUL", "MUFU"]


def main(tag):
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                         check=True).stdout
    fn, counts, total = None, {}, collections.Counter()
    for ln in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]+)?", ln)
        if fn and m:
            op = m.group(2)
            counts[fn]["instr"] += 1
            for k in KEYS:
                if op == k or (op.startswith(k) and k in ("SYNCS", "BAR", "SHFL", "MUFU")):
                    counts[fn][k] += 1
    demangled = {}
    try:
        names = list(counts)
        dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                            check=True).stdout.splitlines()
        demangled = dict(zip(names, dm))
    except Exception:
        pass
    rows = []
    for fn, c in counts.items():
        name = demangled.get(fn, fn)
        name = re.sub(r"ocn::\(anonymous namespace\)::|\(anonymous namespace\)::|ocn::", "", name)
        name = re.sub(r"\(.*", "", name)
        rows.append((name, c))
    rows.sort(key=lambda r: r[0])
    path = os.path.join(ROOT, "profiles", f"sass_summary_{tag}.txt")
    with open(path, "w") as f:
        f.write(f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)} (sm_100a), per kernel\n")
        f.write("# kernel".ljust(60) + "".join(k.rjust(8) for k in ["instr"] + KEYS) + "\n")
        for name, c in rows:
            f.write(name[:59].ljust(60) + "".join(str(c[k]).rjust(8) for k in ["instr"] + KEYS) + "\n")
    print(path, len(rows), "kernels")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
