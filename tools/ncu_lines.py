"""Attribute an ncu SASS source page (per-instruction stall samples) to CUDA source lines.

python tools/ncu_lines.py <report.ncu-rep> [top]   (run here, not on the GPU box)

The line table comes from `nvdisasm --print-line-info` of the in-tree library's cubin (built
with -lineinfo); instruction i of the ncu page is instruction i of the disassembly.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("RMPC_B200_LIB") or os.path.join(ROOT, "paper_2510_12717_b200", "lib", "librmpc_b200.so")
FUNC = os.environ.get("RMPC_NCU_FUNC", "_ZN8rmpc_dev10rti_kernelILb0ELi6EEEvNS_7KParamsE")  # the wide TMEM-only instantiation (T = 9, 10)


def line_table():
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, check=True, capture_output=True)
        # the solve TU's cubin: rmpc_kernel.*, or the device-linked librmpc_b200.* (-rdc=true)
        pre = [os.environ["RMPC_NCU_CUBIN"]] if "RMPC_NCU_CUBIN" in os.environ else ["rmpc_kernel", "librmpc_b200"]
        cub = [f for p in pre for f in sorted(os.listdir(d)) if f.startswith(p + ".") and f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)],
                             check=True, capture_output=True, text=True).stdout
    cur, out, inside = None, [], False
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = ln.startswith(".text." + FUNC + ":")
            continue
        if not inside:
            continue
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
        elif re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
            out.append(cur)
    return out


def functions(path):
    """(first line, name) of every function / lambda-holding definition in a source file."""
    out = []
    for n, ln in enumerate(open(path).read().splitlines(), 1):
        m = re.match(r"(?:template <[^>]*>\s*)?(?:__global__|__device__|__host__)[^(]*?\b(\w+)\(", ln)
        if m:
            out.append((n, m.group(1)))
        m = re.match(r"\s+auto (\w+) = \[", ln)
        if m:
            out.append((n, "lambda:" + m.group(1)))
    return out


def func_of(table, n):
    name = "?"
    for first, f in table:
        if first > n:
            break
        name = f
    return name


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    cs, ci = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    cw, cx = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")
    ins = []
    for r in rows[hi + 1:]:  # the kernel's own table (the page may list called functions after it)
        if r and r[0] == "Address":
            break
        if len(r) > ci:
            ins.append(r)
    lines = line_table()
    if len(lines) != len(ins):
        print(f"warning: {len(ins)} ncu instructions vs {len(lines)} disassembled", file=sys.stderr)
    samp, inst = collections.Counter(), collections.Counter()
    wav, wex = collections.Counter(), collections.Counter()
    for k, r in enumerate(ins):
        key = lines[k] if k < len(lines) else ("?", 0)
        samp[key] += float(r[cs] or 0)
        inst[key] += float(r[ci] or 0)
        wav[key] += float(r[cw] or 0)
        wex[key] += float(r[cx] or 0)
    ts, ti = sum(samp.values()), sum(inst.values())
    csrc = os.path.join(ROOT, "paper_2510_12717_b200", "csrc")
    tables = {f: functions(os.path.join(csrc, f)) for f in os.listdir(csrc) if f.endswith((".cu", ".cuh"))}
    fs, fi = collections.Counter(), collections.Counter()
    for (f, n), v in samp.items():
        key = f"{f}:{func_of(tables[f], n)}" if f in tables else f
        fs[key] += v
        fi[key] += inst[(f, n)]
    print("by function (innermost source function after inlining):")
    for key, v in fs.most_common(30):
        print(f"{100 * v / ts:5.1f}% samp {100 * fi[key] / ti:5.1f}% inst  {key}")
    src = {}
    tw, tx = sum(wav.values()), sum(wex.values())
    print(f"shared wavefronts {tw:.0f}, excessive {tx:.0f} ({100 * tx / max(tw, 1):.1f}%); top lines by excess:")
    for key, v in wex.most_common(12):
        f, n = key
        print(f"  {100 * v / max(tx, 1):5.1f}% of excess, {wav[key]:.0f} wavefronts  {f}:{n}")
    print(f"total samples {ts:.0f}, warp-instructions {ti:.0f}")
    for key, s in samp.most_common(top):
        f, n = key
        if f not in src:
            p = os.path.join(ROOT, "paper_2510_12717_b200", "csrc", f)
            src[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = src[f][n - 1].strip()[:90] if 0 < n <= len(src[f]) else ""
        print(f"{100 * s / ts:5.1f}% samp {100 * inst[key] / ti:5.1f}% inst  {f}:{n}  {text}")


if __name__ == "__main__":
    main()
