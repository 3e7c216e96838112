"""Per-source-line profile of one kernel in an ncu report: the SASS page's executed
instructions, stall samples and shared-memory wavefronts, attributed to CUDA source lines
through the line table of the locally built library (nvdisasm -g; same .so as on the box).

Usage: python tools/ncu_lines.py REPORT.ncu-rep CUBIN_STEM [min_share]
  CUBIN_STEM: the compilation unit (fillblk, merge, commute, ...).
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("PCG_LIB", os.path.join(ROOT, "paper_2401_06713_b200", "libpicasso_b200.so"))


def line_table(stem, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    cub = glob.glob(os.path.join(tmp, stem + ".*.cubin"))[0]
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    funcs, cur, line = {}, None, None
    for ln in out.splitlines():
        m = re.match(r"^(_Z\S+):$", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = {}
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m and cur:
            funcs[cur][int(m.group(1), 16)] = (line, m.group(2))
    return funcs


def main():
    rep, stem = sys.argv[1], sys.argv[2]
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    kname = next(csv.reader([raw[0]]))[1]
    rows = list(csv.reader(raw[1:]))
    h = rows[0]
    ia, ie, ist = h.index("Address"), h.index("Instructions Executed"), h.index(
        "Warp Stall Sampling (All Samples)")
    iw = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
    iwi = h.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in h else None
    rows = [r for r in rows[1:] if len(r) == len(h)]
    base = int(rows[0][ia], 16)
    funcs = line_table(stem, kname)
    # the function whose SASS matches the report's instruction text best
    sass = [(int(r[ia], 16) - base, r[1].strip()) for r in rows]

    norm = lambda x: re.sub(r"0x[0-9a-f]+|`\(\.L_x_\d+\)", "", x).split()

    def score(f):
        t = funcs[f]
        return sum(1 for off, s in sass if off in t and norm(t[off][1]) == norm(s))

    best = max(funcs, key=score)
    table = funcs[best]
    agg = collections.OrderedDict()
    tot_i = tot_s = tot_w = tot_wi = 0
    for r in rows:
        off = int(r[ia], 16) - base
        line = table.get(off, ("?", ""))[0]
        a = agg.setdefault(line, [0, 0, 0, 0])
        i, s = int(r[ie] or 0), int(r[ist] or 0)
        w = int(r[iw] or 0) if iw is not None and r[iw] not in ("", "-") else 0
        wi = int(r[iwi] or 0) if iwi is not None and r[iwi] not in ("", "-") else 0
        a[0] += i; a[1] += s; a[2] += w; a[3] += wi
        tot_i += i; tot_s += s; tot_w += w; tot_wi += wi
    print(f"kernel: {kname}\nfunction: {best}")
    print(f"instructions {tot_i:,}  stall samples {tot_s:,}  smem wavefronts {tot_w:,} "
          f"(ideal {tot_wi:,}, excess {100 * (tot_w - tot_wi) / max(tot_w, 1):.1f}%)")
    print(f"{'line':>18} {'instr%':>7} {'stall%':>7} {'smem wf':>12} {'excess':>10}")
    key = lambda x: int(x[0].split(":")[1]) if ":" in x[0] else 1 << 30
    for line, (i, s, w, wi) in sorted(agg.items(), key=key):
        if i > thr * tot_i or s > thr * tot_s or w > thr * tot_w:
            print(f"{line:>18} {100 * i / tot_i:7.2f} {100 * s / max(tot_s, 1):7.2f} {w:12,} {w - wi:10,}")


if __name__ == "__main__":
    main()
