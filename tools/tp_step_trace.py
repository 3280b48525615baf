"""Where the peer-memory TP reductions of a training step spend their time (MALLEUS_TP_TRACE=1).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/tp_step_trace.py
C2, one TP-2 stage (even plan), 3 warm-up + 2 traced steps.  Per reduction: wait for every member's
ready flag (partner skew), own rows reduced and pushed (last CTA), wait for every member's done."""
import ctypes as C
import os
import sys

os.environ["MALLEUS_TP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from synth.gen import C2_7B_SLICE, make_weights, make_tokens
from paper_2410_13333_b200 import plans as Pl
from paper_2410_13333_b200 import _lib as L
from paper_2410_13333_b200.engine import Engine

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
cfg, B = C2_7B_SLICE, 16
plan = Pl.ladder_plan(cfg, world, B, b=1, straggle=False)
eng = Engine(cfg, rank, world, local)
eng.apply(plan)
eng.write_weights(make_weights(cfg, parity=False))
tok, tgt = make_tokens(cfg, B)
dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
for step in range(1, 6):
    eng.train_step(dtok, dtgt, step=step, apply_update=2)
torch.cuda.synchronize()
L.lib.malleus_k_tp_trace_buffer.restype = C.c_void_p
addr = L.lib.malleus_k_tp_trace_buffer()
buf = np.ctypeslib.as_array((C.c_uint64 * (4096 * 4)).from_address(addr)).reshape(4096, 4).astype(np.int64)
per_step = 16 * (4 * 4 + 1)
last = 5 * per_step  # epochs 1 .. last
ep = np.arange(last - 2 * per_step + 1, last + 1)
rows = buf[ep % 4096]
pos = (ep - 1) % 17
kind = np.where(pos < 8, np.where(pos % 2 == 0, "RESID_NORM", "RESID"), "SUM")
if rank == 0:
    print(f"rank {rank}: {len(ep)} reductions over 2 steps")
for name in ("RESID_NORM", "RESID", "SUM"):
    sel = rows[kind == name]
    ready = (sel[:, 1] - sel[:, 0]) / 1e3
    data = (sel[:, 2] - sel[:, 1]) / 1e3
    done = (sel[:, 3] - sel[:, 2]) / 1e3
    tot = (sel[:, 3] - sel[:, 0]) / 1e3
    print(f"rank {rank} {name:10s} n={len(sel):3d}: ready-wait med {np.median(ready):6.1f} us | rows+push med "
          f"{np.median(data):6.1f} | done-wait med {np.median(done):6.1f} | total med {np.median(tot):6.1f} "
          f"mean {tot.mean():6.1f} us", flush=True)
eng.close()
dist.destroy_process_group()
