"""Two-rank failure scenario for tests/test_gpu_failure.py (torchrun, 2 GPUs):
rank 0 and rank 1 train a C1_MED TP-2 plan (P1) for 2 steps and checkpoint; rank 1 then stops
responding (it skips the next step, like a hung GPU); rank 0's step cannot finish its TP reductions,
its malleus_wait(2 s) returns E_TIMEOUT.  Rank 0 then destroys the context, builds a
1-GPU world, applies plans.survivor_plan (rank 1 at x = infinity), loads the checkpoint
and trains step 3; the loss must equal a fresh single-GPU engine's step 3 from the same checkpoint."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(tmp, out_path):
    from synth.gen import C1_MED, make_weights, make_tokens
    from paper_2410_13333_b200 import plans as Pl
    from paper_2410_13333_b200 import _lib as L
    from paper_2410_13333_b200.engine import Engine
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    cfg, B = C1_MED, 8
    plan = Pl.plan_matrix_c1(cfg, B=B, b=2)["P1"]
    tok, tgt = make_tokens(cfg, B)
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    e = Engine(cfg, rank, world)
    e.apply(plan)
    e.write_weights(make_weights(cfg))
    for s in (1, 2):
        e.train_step(dtok, dtgt, step=s)
    e.wait(10000)
    ck = os.path.join(tmp, "ck")
    e.save_checkpoint(ck, step=2)
    dist.barrier()
    if rank == 1:  # the GPU that stops responding: it never joins step 3 (its process and memory stay
        t = time.time()  # alive until rank 0 is done, so rank 0's peer mappings remain valid)
        while not os.path.exists(out_path) and time.time() - t < 300:
            time.sleep(0.2)
        os._exit(0)
    t0 = time.time()
    status = "ok"
    try:
        e.train_step(dtok, dtgt, step=3)
        e.wait(2000)
    except L.CommTimeout:
        status = "CommTimeout"
    detect_s = time.time() - t0
    e.close()
    # recovery on the surviving GPU: x(rank 1) = infinity -> survivor plan, checkpoint reload
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
    json.dump({"timeout_status": status, "detect_s": detect_s, "survivor_world": len(remap), "loaded_step": step,
               "resumed_loss": resumed, "reference_loss": ref_loss}, open(out_path, "w"))
    os._exit(0)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
