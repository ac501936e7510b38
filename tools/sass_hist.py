"""Static SASS opcode histogram of the in-tree library's kernels (run here; no GPU needed).

python tools/sass_hist.py [kernel-substring ...] > profiles/<tag>_sass_hist.txt

Counts each kernel's static instructions by opcode (cuobjdump -sass): the evidence that the solve
uses TMEM (LDTM/STTM), CUDA-core FP32 (FFMA) and, for the PPO batch, the FP64 tensor cores (DMMA).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("RMPC_SASS_FILE") or os.path.join(ROOT, "paper_2510_12717_b200", "lib", "librmpc_b200.so")
KEEP = ("FFMA", "FMUL", "FADD", "DFMA", "DMUL", "DADD", "DMMA", "HMMA", "UTCMMA", "UTCHMMA", "LDTM", "STTM",
        "LDS", "STS", "LDG", "STG", "LDL", "STL", "SHFL", "BAR", "MUFU", "UBLKCP", "UTMALDG")


def main():
    subs = sys.argv[1:] or ["rti_squad_kernel", "rti_kernel", "rti_shared_kernel", "loss_kernel_mma"]
    txt = subprocess.run(["cuobjdump", "-sass", LIB], check=True, capture_output=True, text=True).stdout
    cur, hist = None, {}
    for ln in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1) if any(s in m.group(1) for s in subs) else None
            if cur:
                hist[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m:
            hist[cur][m.group(2)] += 1
    for fn, h in hist.items():
        tot = sum(h.values())
        print(f"{fn}: {tot} static instructions ({tot * 16 / 1024:.1f} KB)")
        print("  " + "  ".join(f"{k} {h[k]}" for k in KEEP if h[k]))
        print("  top: " + "  ".join(f"{k} {v}" for k, v in h.most_common(12)))


if __name__ == "__main__":
    main()
