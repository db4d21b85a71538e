"""SASS evidence of the built library (no GPU needed): per-function counts of
the instructions that prove tcgen05 / TMA / 256-bit gathers, spill counts,
and the full SASS of the three C4 layer-form kernels' warp-row loops.

  python scripts/sass_evidence.py profiles/r2/sass
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2411_16127_b200", "libgraphfuse_cuda.so")
KEYS = ("UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTMAREDG", "LDTM", "STTM",
        "LDG.E.NA.ELL2.256", "LDG.E.ELL2.256", "LDG.E.NA.ENL2.256", "LDG.E.ENL2.256", "FFMA2", "FMUL2",
        "MUFU.EX2", "STL", "LDL", "R2UR")
# the C4 layer-form kernels (GAT 8x8 fp32: CB 32, LPE 8, CPL 1, VAR GF_ADDV)
MAIN = ("fwd_fastIfLi32ELi8ELi1ELi2ELi0E", "bwd_rows_fastIfLi32ELi8ELi1ELi2E",
        "bwd_cols_fastIfLi32ELi8ELi1ELi2E")


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2", "sass")
    os.makedirs(out, exist_ok=True)
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    with open(os.path.join(out, "mnemonic_counts.txt"), "w") as f:
        f.write("# cuobjdump -sass paper_2411_16127_b200/libgraphfuse_cuda.so (sm_100a; "
                "scripts/sass_evidence.py)\n# per-function counts: tcgen05 / TMA / TMEM, "
                "256-bit gathers (ELL2 = evict_last on the load), paired FMAs, spills\n")
        for name, lines in funcs.items():
            c = collections.Counter()
            for ln in lines:
                ins = re.sub(r"/\*.*?\*/", "", ln).strip()
                op = ins.split(" ;")[0].split()
                if not op:
                    continue
                mn = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
                for k in KEYS:
                    if mn.startswith(k):
                        c[k] += 1
                        break
            if c:
                f.write(f"{name}\n    {dict(sorted(c.items()))}\n")
    for key in MAIN:
        name = next((n for n in funcs if key in n), None)
        if name is None:
            continue
        body = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", ln).rstrip() for ln in funcs[name]]
        body = [ln for ln in body if ln.strip()]
        with open(os.path.join(out, key + ".sass"), "w") as f:
            f.write(f"# full SASS of {name}\n")
            f.write("\n".join(body) + "\n")
    print(out)


if __name__ == "__main__":
    main()
