"""Whole-step parity of the malleable step (libmalleus.so) vs the oracle on the C1 tiny model over
the SURVEY §8(d) plan matrix.  P0 runs in-process on one GPU; multi-GPU plans run under torchrun
with one process per GPU and are skipped when the box has fewer GPUs."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PLAN_WORLD = {"P0": 1, "P1": 2, "P2": 2, "P3": 2, "P4": 4, "P5": 3, "P6": 3, "P7": 8, "P8": 2, "P9": 4,
              "P10": 2, "P11": 4}


def _assert_ok(r):
    assert r["loss_rel"] <= 1e-3, r
    assert r["owned_once"]
    bad = {k: v for k, v in r["grad_rel"].items() if v > 2e-2}
    assert not bad, bad
    bad = {k: v for k, v in r["adam_rel"].items() if v > 1e-6}
    assert not bad, bad
    assert r["push_ok"]
    if "losses" in r:
        for a, b in zip(r["losses"], r["ref_losses"]):
            assert abs(a - b) / abs(b) <= 1e-3, (r["losses"], r["ref_losses"])


def test_p0_single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from tests.mp_worker import run
    r = run("P0", steps=4)
    _assert_ok(r)


def test_p0_single_gpu_d128():
    """C1_MED (d = 128, s = 256, 512-token micro-batches): the tcgen05 attention kernels and the
    CTA-pair GEMM with TMA-store / TMA-reduce-add epilogues run inside the step."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from tests.mp_worker import run
    r = run("P0", steps=3, cfg_name="c1m")
    _assert_ok(r)


@pytest.mark.parametrize("plan", ["P2", "P4", "P9"])
def test_multi_gpu_plans_d128(plan, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = PLAN_WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
           str(out), "2", "c1m"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, "\n".join(l for l in (p.stdout + p.stderr).splitlines()
                                        if "Error" in l or "error" in l or "rank" in l)[-6000:]
    _assert_ok(json.load(open(out)))


@pytest.mark.parametrize("plan", ["P1", "P2", "P3", "P8", "P10", "P5", "P6", "P4", "P9", "P11", "P7"])
def test_multi_gpu_plans(plan, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = PLAN_WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
           str(out), "2"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, "\n".join(l for l in (p.stdout + p.stderr).splitlines()
                                        if "Error" in l or "error" in l or "rank" in l)[-6000:]
    _assert_ok(json.load(open(out)))


def test_tp_peer_reduce_matches_nccl(tmp_path):
    """The fused peer-memory TP reduction (tp_reduce.cu: reduce-scatter + push, fused residual and
    RMSNorm) against the NCCL all-reduce path (MALLEUS_NO_P2P=1) on P2 (TP 2, uneven heads), C1_MED:
    with two members every row sum is one fp32 addition on both paths and the norm arithmetic is
    the same, so with fp32 partials (MALLEUS_TP_PARTIAL=fp32) the losses of a 3-step run must agree
    bit for bit.  (The default bf16 partials are covered by the oracle parity of every TP plan.)"""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = {}
    for tag, extra in (("peer", {"MALLEUS_TP_PARTIAL": "fp32"}), ("nccl", {"MALLEUS_NO_P2P": "1"})):
        out = tmp_path / f"{tag}.json"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr=127.0.0.1", "--master-port=29535", os.path.join(ROOT, "tests", "mp_worker.py"), "P2",
               str(out), "3", "c1m"]
        p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env={**os.environ, **extra})
        assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
        res[tag] = json.load(open(out))
        _assert_ok(res[tag])
    assert res["peer"]["losses"] == res["nccl"]["losses"], (res["peer"]["losses"], res["nccl"]["losses"])


@pytest.mark.parametrize("plan", ["P2", "P9"])
def test_tp_scatter_epilogue_bitwise(plan, tmp_path):
    """Reduce-scatter fused into the row-parallel GEMM epilogue (rows stored straight into the owning
    member's receive slot over NVLink) against the unfused peer path (MALLEUS_TP_NO_SCATTER=1): the
    same bf16 partials summed in the same member order, so a 3-step run's losses agree bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = PLAN_WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    res = {}
    for tag, extra in (("scatter", {"MALLEUS_TP_SCATTER_K": "4"}), ("pull", {"MALLEUS_TP_NO_SCATTER": "1"})):
        out = tmp_path / f"{tag}.json"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", "--master-port=29536", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
               str(out), "3", "c1m"]
        p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env={**os.environ, **extra})
        assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
        res[tag] = json.load(open(out))
        _assert_ok(res[tag])
    assert res["scatter"]["losses"] == res["pull"]["losses"], (res["scatter"]["losses"], res["pull"]["losses"])


@pytest.mark.parametrize("plan", ["P2", "P9"])
def test_wgrad_pair_on_tp_stage(plan, tmp_path):
    """Paired weight-gradient GEMMs (K = 2T over micro-batches 2p, 2p + 1) are on by default only on
    TP-1 single-stage pipelines; MALLEUS_WGRAD_PAIR_TP=1 turns them on for TP > 1 stages too (the
    backward TP sums then overlap the flush micro-batch's GEMMs only): oracle parity of the step."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = PLAN_WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
           str(out), "2", "c1m"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "MALLEUS_WGRAD_PAIR_TP": "1"})
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    _assert_ok(json.load(open(out)))


def test_p0_run_to_run_bitwise():
    """Determinism: every reduction runs in a fixed order (no float atomics; the
    embedding backward sums repeated tokens in position order), so two runs of the same plan give
    bit-identical losses over 3 steps (the later losses depend on every gradient through AdamW)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from tests.mp_worker import run
    a = run("P0", steps=3)
    b = run("P0", steps=3)
    assert a["losses"] == b["losses"], (a["losses"], b["losses"])


@pytest.mark.parametrize("plan", ["P0", "P4"])
def test_grad_clipping(plan, tmp_path, monkeypatch):
    """Global-norm gradient clipping (malleus_adam_cfg.max_grad_norm, torch clip_grad_norm_
    semantics): the norm the library computes from the owners' reduced gradients equals the norm
    of the gathered reduced gradients, the update equals the oracle's AdamW on the clipped gradient,
    and a 3-step loss curve follows the oracle trained with clipping.  max_grad_norm is set below
    the step-1 norm so clipping is active."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = PLAN_WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    monkeypatch.setenv("MALLEUS_TEST_CLIP", "0.05")
    if n == 1:
        from tests.mp_worker import run
        r = run(plan, steps=3)
    else:
        out = tmp_path / "r.json"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
               str(out), "3"]
        p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=dict(os.environ))
        assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
        r = json.load(open(out))
    _assert_ok(r)
    assert r["clip_coef"] < 1.0, r["clip_coef"]  # clipping was active
    assert abs(r["grad_norm"] - r["grad_norm_rgrad"]) <= 1e-4 * r["grad_norm_rgrad"], (r["grad_norm"], r["grad_norm_rgrad"])
