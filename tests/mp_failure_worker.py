"""Failure scenario for tests/test_gpu_failure.py.

detect (torchrun, 2 GPUs): both ranks train a C1_MED TP-2 plan (P1) for 2 steps and checkpoint; then
  rank 1 stops responding (it never joins step 3, like a hung GPU; its process stays alive so rank
  0's peer mappings stay valid until rank 0 is done).  Rank 0 enqueues step 3, whose TP reductions
  wait for rank 1, and malleus_wait(2 s) must return E_TIMEOUT.  Rank 0 records the
  outcome and exits: the job ends, as a failed training job does.
recover (one process, the surviving GPU): the job restarts on GPU 0 with rank 1's straggling rate
  set to infinity (plans.survivor_plan), loads the checkpoint and trains step 3; the
  loss must equal that of a fresh single-GPU engine trained from the same checkpoint."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def _setup():
    from synth.gen import C1_MED, make_tokens
    from paper_2410_13333_b200 import plans as Pl
    cfg, B = C1_MED, 8
    tok, tgt = make_tokens(cfg, B)
    return cfg, B, Pl.plan_matrix_c1(cfg, B=B, b=2)["P1"], tok, tgt


def detect(tmp):
    import torch.distributed as dist
    from synth.gen import make_weights
    from paper_2410_13333_b200 import _lib as L
    from paper_2410_13333_b200.engine import Engine
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    cfg, B, plan, tok, tgt = _setup()
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    e = Engine(cfg, rank, world)
    e.apply(plan)
    e.write_weights(make_weights(cfg))
    for s in (1, 2):
        e.train_step(dtok, dtgt, step=s)
    e.wait(10000)
    e.save_checkpoint(os.path.join(tmp, "ck"), step=2)
    dist.barrier()
    flag = os.path.join(tmp, "detected.json")
    if rank == 1:  # unresponsive from here on
        t = time.time()
        while not os.path.exists(flag) and time.time() - t < 120:
            time.sleep(0.1)
        os._exit(0)
    t0 = time.time()
    status = "ok"
    try:
        e.train_step(dtok, dtgt, step=3)
        e.wait(2000)
    except L.CommTimeout:
        status = "CommTimeout"
    except L.MalleusError as err:  # noqa: F841
        status = "MalleusError"
    json.dump({"timeout_status": status, "detect_s": time.time() - t0,
               "state_after": L.lib.malleus_wait(e.ctx, None, 10)}, open(flag + ".tmp", "w"))
    os.rename(flag + ".tmp", flag)
    os._exit(0)


def recover(tmp, out_path):
    from paper_2410_13333_b200 import plans as Pl
    from paper_2410_13333_b200.engine import Engine
    cfg, B, plan, tok, tgt = _setup()
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    ck = os.path.join(tmp, "ck")
    new_plan, remap = Pl.survivor_plan(cfg, plan, failed=[1])
    s = Engine(cfg, 0, 1, 0)
    s.apply(new_plan)
    step = s.load_checkpoint(ck)
    resumed = s.train_step(dtok, dtgt, step=step + 1).item()
    s.close()
    ref = Engine(cfg, 0, 1, 0)
    ref.apply(Pl.plan_matrix_c1(cfg, B=B, b=2)["P0"])
    ref.load_checkpoint(ck)
    ref_loss = ref.train_step(dtok, dtgt, step=step + 1).item()
    ref.close()
    det = json.load(open(os.path.join(tmp, "detected.json")))
    json.dump(dict(det, survivor_world=len(remap), loaded_step=step, resumed_loss=resumed, reference_loss=ref_loss),
              open(out_path, "w"))


if __name__ == "__main__":
    if sys.argv[1] == "detect":
        detect(sys.argv[2])
    else:
        recover(sys.argv[2], sys.argv[3])
