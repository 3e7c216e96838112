"""Static SASS opcode mix of the shipped default kernels (cuobjdump -sass on the built library).

Usage: python tools/sass_mix.py > profiles/r2_sass_mix.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2401_06713_b200", "libpicasso_b200.so")
DEFAULT = ["k_commute_fr8", "k_commute_direct", "k_owned_fr", "k_count_owned", "k_fill_blk", "k_fill_bins", "k_delta",
           "k_encode", "k_lists", "k_bucket_bounds", "k_compact"]
SHOW = 12
KEY = {"LDS", "STS", "POPC", "PRMT", "ATOMS", "REDS", "RED", "LDG", "STG", "BAR", "SHFL", "FLO"}


def main():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True,
                          text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            op = m.group(2) + (m.group(3) or "")
            funcs[cur][op] += 1
    print("Static SASS opcode mix (cuobjdump -sass libpicasso_b200.so), sm_100a, round-2 build.")
    print("Shipped default kernels only. No HMMA/UTC*MMA: the path is bitwise integer work")
    print("(LOP3/POPC/PRMT + shared-memory tables); the fills are shared-memory bitmaps/bins.\n")
    for k in DEFAULT:
        names = sorted(f for f in funcs if re.search(r"\d" + k + r"I|\d" + k + r"E", f))
        for f in names:
            c = funcs[f]
            print(f"{f}  ({sum(c.values())} instructions)")
            top = c.most_common(SHOW)
            key = [(op, cnt) for op, cnt in sorted(c.items()) if op.split(".")[0] in KEY
                   and (op, cnt) not in top]
            for op, cnt in top + key:
                print(f"   {op:28s} {cnt}")
            mma = [op for op in c if op.startswith(("HMMA", "UTC", "IMMA"))]
            tma = [op for op in c if op.startswith(("UBLKCP", "UTMALDG", "UTMASTG", "SYNCS"))]
            print(f"   tensor-core ops: {mma or 'none'}; bulk-copy/TMA ops: {tma or 'none'}\n")


if __name__ == "__main__":
    main()
