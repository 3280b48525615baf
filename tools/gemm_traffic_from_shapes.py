"""roofline.traffic source for bench.py: DRAM bytes per GEMM launch of one C2 N = 1 step, measured by ncu
(dram__bytes_read.sum + dram__bytes_write.sum of every gemm_tcgen05 launch of the step, the same capture
tools/gemm_shapes_report.py tabulates per shape), against the algorithmic bytes of the same launches.

  python tools/gemm_traffic_from_shapes.py shapes.csv gemm_log.txt SKIP > profiles/gemm_traffic.json
"""
import csv
import json
import sys
from collections import OrderedDict


def main(csv_path, log_path, skip):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kid, kn, mn, mv, mu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1.0, "B": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9,
             "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "%": 1.0}
    per = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > mv and "gemm_tcgen05" in r[kn]:
            per.setdefault(r[kid], {})[r[mn]] = float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
    launches = list(per.values())
    log = [l.split() for l in open(log_path).read().splitlines()][skip: skip + len(launches)]
    rd = sum(m.get("dram__bytes_read.sum", 0.0) for m in launches)
    wr = sum(m.get("dram__bytes_write.sum", 0.0) for m in launches)
    t = sum(m.get("gpu__time_duration.sum", 0.0) for m in launches)
    alg = 0.0
    for l in log:
        M, N, K, _, _, mode, epi = (int(x) for x in l[:7])
        csz = 2 if mode == 0 else 4
        a = (M * K + K * N) * 2 + M * N * csz * (2 if mode == 2 else 1)
        if epi == 1:
            a += M * (N // 2) * 2
        elif epi == 2:
            a += M * N * 2 * 3 - M * N * 2
        elif epi == 3:
            a += M * N * 2
        alg += a
    n = len(launches)
    print(json.dumps({"kernel": "gemm_tcgen05 (all GEMM launches of one C2 N=1 step)", "launches": n,
                      "bytes_per_launch": (rd + wr) / n, "dram_read_bytes_per_launch": rd / n,
                      "dram_write_bytes_per_launch": wr / n, "algorithmic_bytes_per_launch": alg / n,
                      "traffic_over_algorithmic": (rd + wr) / alg, "ncu_gemm_seconds_per_step": t,
                      "source": csv_path}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]))
