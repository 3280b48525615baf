"""DRAM traffic of the step's GEMM launches vs their algorithmic bytes (bench.py `roofline.traffic`).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm \
      --csv --log-file gemm_dram.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline
  python tools/gemm_traffic.py gemm_dram.csv > profiles/gemm_traffic.json

The last step's launches (816 GEMMs at C2, N = 1: 4 layers x 16 micro-batches x 12 + 3 LM-head GEMMs
x 16) are summed.  Algorithmic bytes per GEMM: A and B read once (bf16), C written once (bf16 or
fp32), and for the fp32 weight-gradient accumulation (every micro-batch after the first) C read
and written once (the tensors exceed L2)."""
import csv
import json
import sys
from collections import OrderedDict


def c2_algorithmic_bytes():
    T, h, nd, F, V, L, M = 2048, 4096, 4096, 11008, 32000, 4, 16
    tot, n = 0, 0

    def g(m, nn, k, out_b, acc=False):
        nonlocal tot, n
        tot += 2 * (m * k + nn * k) + (8 if acc else out_b) * m * nn
        n += 1
    for mb in range(M):
        acc = mb > 0
        for _ in range(L):
            g(T, 3 * nd, h, 2); g(T, h, nd, 4); g(T, 2 * F, h, 2); g(T, h, F, 4)       # forward
            g(T, F, h, 2); g(F, h, T, 4, acc); g(T, h, 2 * F, 4); g(2 * F, h, T, 4, acc)  # MLP backward
            g(T, nd, h, 2); g(nd, h, T, 4, acc); g(T, h, 3 * nd, 4); g(3 * nd, h, T, 4, acc)  # attention bwd
        g(T, V, h, 4); g(T, h, V, 4); g(V, h, T, 4, acc)                                  # LM head
    return tot, n


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    iid, kn, mn, mv, mu = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= mv or "gemm" not in r[kn]:
            continue
        v = float(r[mv].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(r[mu], 1)
        launches.setdefault(r[iid], {})[r[mn]] = v * scale
    alg, per_step = c2_algorithmic_bytes()
    last = list(launches.values())[-per_step:]
    rd = sum(x.get("dram__bytes_read.sum", 0) for x in last)
    wr = sum(x.get("dram__bytes_write.sum", 0) for x in last)
    t = sum(x.get("gpu__time_duration.sum", 0) for x in last)
    print(json.dumps({
        "kernel": "gemm_tcgen05 (all GEMM launches of one C2 N=1 step)",
        "launches": len(last),
        "bytes_per_launch": (rd + wr) / len(last),
        "dram_read_bytes_per_launch": rd / len(last),
        "dram_write_bytes_per_launch": wr / len(last),
        "algorithmic_bytes_per_launch": alg / per_step,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "ncu_gemm_seconds_per_step": t,
        "source": path,
    }, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
