"""Per-shape GEMM evidence of one training step: joins an ncu metrics list of the
gemm_tcgen05 launches with the MALLEUS_GEMM_LOG shape log of the same program (n-th launch <-> n-th
line after `skip`) and aggregates per (M, N, K, layouts, epilogue): launches, mean ncu time, TF/s,
tensor-pipe active % (sm__pipe_tensor_cycles_active, % of peak sustained active) and DRAM bytes vs
the algorithmic bytes (A + B read once, C written once; fp32 accumulate epilogues read + write C).

  MALLEUS_GEMM_LOG=log.txt ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:gemm_tcgen05 --launch-skip S --launch-count N --csv --log-file m.csv python bench.py ...
  python tools/gemm_shapes_report.py m.csv log.txt S > profiles/r02/gemm_shapes.md
"""
import csv
import sys
from collections import OrderedDict, defaultdict

EPI = {0: "plain", 1: "+SwiGLU", 2: "+SwiGLU-bwd", 3: "+residual"}
MODE = {0: "bf16", 1: "f32", 2: "f32+="}


def main(csv_path, log_path, skip):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kid, kn, mn, mv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    mu = h.index("Metric Unit")
    scale = {"byte": 1.0, "B": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9,
             "nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "%": 1.0}
    per = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= mv or "gemm_tcgen05" not in r[kn]:
            continue  # bytes and ns after scaling
        per.setdefault(r[kid], {})[r[mn]] = float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
    launches = list(per.values())
    log = [l.split() for l in open(log_path).read().splitlines()][skip: skip + len(launches)]
    assert len(log) == len(launches), (len(log), len(launches))
    agg = defaultdict(lambda: defaultdict(float))
    for m, l in zip(launches, log):
        M, N, K, amn, bmn, mode, epi = (int(x) for x in l[:7])
        key = (M, N, K, amn, bmn, mode, epi)
        a = agg[key]
        a["n"] += 1
        a["t"] += m.get("gpu__time_duration.sum", 0.0)
        a["tc"] += m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    tot_t = sum(a["t"] for a in agg.values())
    print(f"# GEMM shapes of one step ({len(launches)} launches, ncu, {csv_path})\n")
    print("| M | N | K | A,B layout | C | epilogue | launches | mean us | TF/s | tensor-pipe active % | DRAM MB / algorithmic MB | share of GEMM time |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for (M, N, K, amn, bmn, mode, epi), a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        n = a["n"]
        t_us = a["t"] / n / 1e3  # ncu reports ns
        tf = 2.0 * M * N * K / (t_us * 1e-6) / 1e12
        csz = 2 if mode == 0 else 4
        alg = (M * K + K * N) * 2 + M * N * csz * (2 if mode == 2 else 1)
        if epi == 1:
            alg += M * (N // 2) * 2
        elif epi == 2:
            alg += M * N * 2 * 2 + M * N * 2 * 2 - M * N * 2  # reads gu, writes dgu, no du
        elif epi == 3:
            alg += M * N * 2
        dram = (a["rd"] + a["wr"]) / n
        print(f"| {M} | {N} | {K} | {'MN' if amn else 'K'},{'MN' if bmn else 'K'} | {MODE[mode]} | {EPI.get(epi, epi)} | "
              f"{n:.0f} | {t_us:.1f} | {tf:.0f} | {a['tc'] / n:.1f} | {dram / 1e6:.1f} / {alg / 1e6:.1f} | "
              f"{a['t'] / tot_t:.1%} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
