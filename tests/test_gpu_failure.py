"""Failure path.

* Detection: the device-side communication waits of the peer-memory TP reduction give up when a
  member never arrives — released by the process-wide abort word (what malleus_wait sets on its
  timeout) or by their own timeout (MALLEUS_COMM_TIMEOUT_MS) — instead of hanging or trapping; the
  status word reports it and the device stays usable (single GPU: co-resident members, one absent).
* Recovery: a checkpoint of the owned ZeRO-1 pieces (Engine.save_checkpoint) restores bit for bit
  into a fresh context, also under another plan, and training continues identically.
* End to end (2 GPUs): rank 1 stops responding in the middle of a TP-2 step; rank 0's malleus_wait
  returns E_TIMEOUT, and rank 0 resumes alone from the last checkpoint with rank 1's rate set to
  infinity (plans.survivor_plan), matching a single-GPU run from the same checkpoint."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_13333_b200 import _lib
    return _lib


def _wait_stream(stream, seconds):
    t0 = time.time()
    while not stream.query():
        if time.time() - t0 > seconds:
            return False
        time.sleep(0.005)
    return True


def test_tp_reduce_absent_member_released_by_abort(L):
    from tests.tputil import Group
    L.lib.malleus_k_comm_abort(0)
    L.lib.malleus_k_comm_status(1)
    G = Group(2, 128, 512, devices=[0, 0])
    G.launch(0, skip={1})  # member 1 never arrives
    assert not _wait_stream(G.streams[0], 0.3)  # member 0 is waiting for it
    assert L.lib.malleus_k_comm_status(0) == 0
    L.lib.malleus_k_comm_abort(1)  # malleus_wait's failure path
    assert _wait_stream(G.streams[0], 10.0), "the abort word did not release the wait"
    assert L.lib.malleus_k_comm_status(1) == 1
    L.lib.malleus_k_comm_abort(0)
    torch.cuda.synchronize()
    # the device is healthy: a complete reduction on fresh buffers is exact
    G2 = Group(2, 128, 512, devices=[0, 0])
    for j in range(2):
        G2.part[1][j].copy_(torch.full((128, 512), float(j + 1), device="cuda"))
    G2.launch(0)
    G2.sync()
    assert torch.equal(G2.out32[0], torch.full((128, 512), 3.0, device="cuda"))
    assert L.lib.malleus_k_comm_status(0) == 0


def test_tp_reduce_absent_member_times_out():
    """Without an abort, the wait gives up by itself after MALLEUS_COMM_TIMEOUT_MS (fresh process)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    code = (
        "import time, torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2410_13333_b200 import _lib as L\n"
        "from tests.tputil import Group\n"
        "G = Group(2, 128, 512, devices=[0, 0]); t = time.time(); G.launch(0, skip={1}); G.sync()\n"
        "print(L.lib.malleus_k_comm_status(1), round(time.time() - t, 2))\n" % ROOT)
    env = dict(os.environ, MALLEUS_COMM_TIMEOUT_MS="400")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    status, secs = out.stdout.split()[-2:]
    assert int(status) == 1 and 0.3 <= float(secs) < 30, out.stdout


def _engine(cfg, plan):
    from paper_2410_13333_b200.engine import Engine
    e = Engine(cfg, 0, 1, 0)
    e.apply(plan)
    return e


def _state(e, cfg):
    from paper_2410_13333_b200 import _lib as Lb
    from paper_2410_13333_b200.engine import tensor_names
    out = {}
    for n in tensor_names(cfg):
        for k in (Lb.KIND_PARAM, Lb.KIND_MASTER, Lb.KIND_ADAM_M, Lb.KIND_ADAM_V):
            r, v = e.read(n, k)
            out[(n, k)] = (r, v.copy())
    return out


def test_checkpoint_roundtrip_bitwise(L, tmp_path):
    from synth.gen import C1_MED, make_weights, make_tokens
    from paper_2410_13333_b200 import plans as Pl
    cfg, B = C1_MED, 8
    plan = Pl.plan_matrix_c1(cfg, B=B, b=2)["P0"]
    tok, tgt = make_tokens(cfg, B)
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    e = _engine(cfg, plan)
    e.write_weights(make_weights(cfg))
    for s in (1, 2):
        e.train_step(dtok, dtgt, step=s)
    e.save_checkpoint(str(tmp_path / "ck"), step=2)
    ref_state = _state(e, cfg)
    loss3 = e.train_step(dtok, dtgt, step=3).item()
    after3 = _state(e, cfg)
    e.close()
    f = _engine(cfg, plan)
    assert f.load_checkpoint(str(tmp_path / "ck")) == 2
    st = _state(f, cfg)
    for key, (r, v) in ref_state.items():
        assert st[key][0] == r and np.array_equal(st[key][1], v), key
    assert f.train_step(dtok, dtgt, step=3).item() == loss3
    st3 = _state(f, cfg)
    for key, (r, v) in after3.items():
        assert np.array_equal(st3[key][1], v), key
    f.close()
    # another plan (micro-batch 1 instead of 2): the same logical state is loaded
    g = _engine(cfg, Pl.plan_matrix_c1(cfg, B=B, b=1)["P0"])
    g.load_checkpoint(str(tmp_path / "ck"))
    st = _state(g, cfg)
    for key, (r, v) in ref_state.items():
        assert np.array_equal(st[key][1], v), key
    g.close()


def _run_group(cmd, timeout):
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT,
                         start_new_session=True)
    try:
        so, se = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:  # kill the whole process group (torchrun and its workers)
        os.killpg(p.pid, 9)
        so, se = p.communicate()
    return p.returncode, so, se


def test_failure_detected_and_survivor_resumes(tmp_path):
    """2 GPUs: TP2 plan; rank 1 hangs; rank 0 detects it (E_TIMEOUT, then E_STATE); the job restarts
    on GPU 0 alone from the checkpoint with rank 1 at x = infinity."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    worker = os.path.join(ROOT, "tests", "mp_failure_worker.py")
    rc, so, se = _run_group([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                             "--master-addr=127.0.0.1", "--master-port=29541", worker, "detect", str(tmp_path)], 240)
    assert (tmp_path / "detected.json").exists(), so[-3000:] + se[-3000:]
    out = tmp_path / "r.json"
    rc, so, se = _run_group([sys.executable, worker, "recover", str(tmp_path), str(out)], 240)
    assert out.exists(), so[-3000:] + se[-3000:]
    r = json.loads(out.read_text())
    assert r["timeout_status"] == "CommTimeout", r
    assert r["detect_s"] < 30 and r["state_after"] == 6, r  # MALLEUS_E_STATE: the context is failed
    assert r["survivor_world"] == 1 and r["loaded_step"] == 2
    assert r["resumed_loss"] == r["reference_loss"], r
