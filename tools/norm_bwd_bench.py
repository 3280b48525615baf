"""RMSNorm backward kernel A/B at the C2 shape (T = 2048, h = 4096, bf16 dy, residual gradient):
the row-group kernel (default), the block kernel (MALLEUS_NORM_BWD_BLOCK=1) and the warp-per-row
kernel (MALLEUS_NORM_BWD_WARP=1), each in its own process (the switches are read once).  Times one
malleus_k_rmsnorm_bwd16 call (norm kernel + colsum pass) with CUDA events, L2-hot (the same buffers
every call: in the step the operands were just written by the producing GEMM) and L2-cold (rotating
over 6 buffer sets, 400 MB > the 126 MB L2).  HBM bytes per call: x, dy, dres read, dx written.

  python tools/norm_bwd_bench.py            # runs the three variants
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(T=2048, h=4096, reps=200):
    import torch
    from paper_2410_13333_b200 import _lib as L
    torch.manual_seed(0)
    sets = []
    for _ in range(6):
        sets.append(dict(x=torch.randn(T, h, device="cuda").bfloat16(), dy=torch.randn(T, h, device="cuda").bfloat16(),
                         dres=torch.randn(T, h, device="cuda").bfloat16(), dx=torch.empty(T, h, device="cuda").bfloat16()))
    g = (1 + 0.1 * torch.randn(h, device="cuda")).bfloat16()
    r = torch.rand(T, device="cuda") + 0.5
    dg = torch.zeros(h, device="cuda")
    st = torch.cuda.current_stream()

    def call(b):
        rc = L.lib.malleus_k_rmsnorm_bwd16(T, h, b["x"].data_ptr(), g.data_ptr(), r.data_ptr(), b["dy"].data_ptr(),
                                           b["dres"].data_ptr(), b["dx"].data_ptr(), dg.data_ptr(), st.cuda_stream)
        assert rc == 0

    out = {}
    for mode in ("hot", "cold"):
        for i in range(10):
            call(sets[0])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(reps):
            call(sets[0] if mode == "hot" else sets[i % 6])
        b.record(st)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / reps * 1e3
        out[mode] = {"us": round(us, 2), "GBps": round(4 * T * h * 2 / (us * 1e-6) / 1e9, 1)}
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        print(json.dumps(one()))
        sys.exit(0)
    res = {}
    for name, env in (("rows (default)", {}), ("block", {"MALLEUS_NORM_BWD_BLOCK": "1"}),
                      ("warp", {"MALLEUS_NORM_BWD_WARP": "1"})):
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--one"], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=600)
        res[name] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-500:]
        print(name, res[name], flush=True)
    print(json.dumps({"shape": "T 2048, h 4096, bf16 dy + dres", "includes": "norm kernel + colsum_accum + "
                      "cudaMallocAsync/FreeAsync of the scratch (k_ entry point)", "results": res}))
