"""HBM / NVLink roofline table for the non-GEMM kernels of a C2 N = 1 step (SURVEY §8(d) "which
roofline bounds what"): achieved GB/s = algorithmic bytes per launch / mean ncu launch time
(cold-cache, serialised: a lower bound on the in-step rate), against the measured 6550 GB/s.

  python tools/hbm_report.py profiles/r02/launches_c2_n1_final.csv > profiles/r02/hbm_roofline.md
"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

T, h, F, V, nd = 2048, 4096, 11008, 32000, 4096
P_TOTAL = 4 * (4 * h * h + 3 * h * F) + 2 * V * h + 9 * h  # C2 slice parameters (1.07 B)
# algorithmic bytes per launch (reads + writes), C2 shapes at N = 1
ALG = {
    # round 2 (TP 1): the residual adds are fused into the O / down GEMM epilogues, so the forward
    # norm reads x1 (bf16) and writes a (bf16); the backward norm reads a bf16 dy
    "rmsnorm_fwd_kernel": ("x bf16 in, a bf16 out (+ rstd)", (2 + 2) * T * h + 4 * T),
    "rmsnorm_bwd_warp_kernel": ("x, dy, dres bf16 in, dx bf16 out (+ 148 x h fp32 dg partials)",
                                (2 + 2 + 2 + 2) * T * h + 4 * 148 * h),
    "rmsnorm_bwd_kernel": ("x, dres, dx bf16 + dy fp32 (+ 888 x h fp32 dg partials)", (2 + 2 + 2 + 4) * T * h + 4 * 888 * h),
    "colsum_accum_kernel": ("148 x h fp32 CTA partials (warp kernel)", 4 * 148 * h),
    "swiglu_fwd_kernel": ("gu bf16 in, u bf16 out", 2 * T * 2 * F + 2 * T * F),
    "swiglu_bwd_kernel": ("gu, du in, dgu out (bf16)", 2 * T * 2 * F + 2 * T * F + 2 * T * 2 * F),
    "ce_stats_kernel": ("logits fp32", 4 * T * V),
    "ce_grad_kernel": ("logits fp32 in, dlogits bf16 out", 4 * T * V + 2 * T * V),
    "reduce_adam_kernel": ("30 B per parameter (grad, master, m, v in; master, m, v, bf16 param out)", 30 * P_TOTAL),
    "attn_dsum_kernel": ("O, dO bf16", 2 * 2 * T * nd),
    "residual_add_kernel": ("x bf16 + partial fp32 in, bf16 out", (2 + 4 + 2) * T * h),
    "embed_bwd_kernel": ("dx bf16 in, dE rows fp32 read-modify-write", 2 * T * h + 8 * T * h),
}


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name).replace("mls::", "").replace("(anonymous namespace)::", "")
    name = name.replace("<unnamed>::", "")
    name = re.sub(r"<.*>", "", name)
    return name.strip()


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    kn, mn, mv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mv and r[mn] == "gpu__time_duration.sum":
            agg[short(r[kn])].append(float(r[mv].replace(",", "")) * 1e-9)
    peak = 6550.1
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peak = json.load(open(mp)).get("hbm_gbs", peak)
    print(f"# HBM roofline of the non-GEMM kernels (C2, N = 1; `{path}`)\n")
    print(f"Peak: {peak:.0f} GB/s (MEASURED_PEAKS.json copy bandwidth). Times are ncu cold-cache serialised means.\n")
    print("| kernel | launches | mean us | algorithmic MB / launch | GB/s | of peak | bytes counted |")
    print("|---|---|---|---|---|---|---|")
    for k, (what, b) in ALG.items():
        ts = agg.get(k)
        if not ts:
            continue
        t = sum(ts) / len(ts)
        print(f"| `{k}` | {len(ts)} | {t*1e6:.1f} | {b/1e6:.1f} | {b/t/1e9:.0f} | {b/t/1e9/peak:.0%} | {what} |")


if __name__ == "__main__":
    main(sys.argv[1])
