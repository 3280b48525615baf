"""A whole C2 step of the CPU oracle, timed once (VERDICT r1 "measurement hygiene": the bench's
cpu_baseline extrapolates from one 2048-token sequence through 1 of the 4 layers; this checks that
extrapolation against the full workload on the same host).

The full step is the oracle's forward + backward of all B = 16 sequences of 2048 tokens through the
embedding, the 4 layers and the LM head (numpy fp64, `oracle.model.forward_backward`), one sequence
per call (the per-sequence attention matrices of a 16-sequence call would need ~70 GB; the step's
gradient is the sum of the per-sequence gradients, so the arithmetic is the same).  AdamW is not
timed (a few elementwise passes over 1.1 B parameters, negligible next to the GEMMs).

  python tools/oracle_full_step.py [--seqs 16] > profiles/r02/oracle_full_step.json
"""
import argparse
import dataclasses
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=16)
    args = ap.parse_args()
    import bench
    from synth.gen import C2_7B_SLICE, make_weights, make_tokens
    from oracle import model as M
    cfg = C2_7B_SLICE
    sample = bench.oracle_sample(cfg, seq=2048, reps=1)  # the bench's estimate on this host
    print(json.dumps({"bench_cpu_baseline_estimate": sample}), file=sys.stderr, flush=True)
    one = dataclasses.replace(cfg)
    P = M.params_f64(make_weights(one))
    tok, tgt = make_tokens(one, args.seqs)
    ts = []
    for i in range(args.seqs):
        t0 = time.perf_counter()
        M.forward_backward(one, P, tok[i:i + 1], tgt[i:i + 1])
        ts.append(time.perf_counter() - t0)
        print(f"sequence {i}: {ts[-1]:.1f} s", file=sys.stderr, flush=True)
    total = sum(ts)
    tokens = args.seqs * cfg.seq_len
    full = tokens / total
    out = {"workload": "C2 (4 layers, h 4096, 32 heads, F 11008, V 32000), %d x %d tokens" % (args.seqs, cfg.seq_len),
           "host_threads": sample["cores"], "full_step_seconds": total, "full_step_tokens_s": full,
           "per_sequence_seconds": {"median": statistics.median(ts), "min": min(ts), "max": max(ts)},
           "bench_estimate_tokens_s": sample["value"], "estimate_over_full": sample["value"] / full,
           "bench_sample": sample["sample"]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
