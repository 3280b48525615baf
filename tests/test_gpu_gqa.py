"""GQA on the GPU path: n_kv = n/2 KV heads, query head j reads KV head
j // g (oracle/model.py).  Whole-step parity against the oracle (readings R15 / R16) on one GPU and on
the GQA plan matrix (TP 2 with whole KV groups per member, cross-layout DP, PP), plus the rejection of
a head split that cuts a KV group.  head_dim 128 runs the tcgen05 attention, head_dim 32 the
mma.sync kernels; FP32 mode the SIMT kernels."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = {"P1": 2, "P3": 2, "P4": 3, "P6": 3}


def _ok(r):
    assert r["loss_rel"] <= 1e-3, r
    assert r["owned_once"]
    bad = {k: v for k, v in r["grad_rel"].items() if v > 2e-2}
    assert not bad, bad
    bad = {k: v for k, v in r["adam_rel"].items() if v > 1e-6}
    assert not bad, bad
    assert r["push_ok"]
    for a, b in zip(r.get("losses", []), r.get("ref_losses", [])):
        assert abs(a - b) / abs(b) <= 1e-3


@pytest.mark.parametrize("cfg_name", ["c1g", "c1mg"], ids=["d32_mma_sync", "d128_tcgen05"])
def test_gqa_p0_single_gpu(cfg_name):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from tests.mp_worker import run
    _ok(run("P0", steps=3, cfg_name=cfg_name))


@pytest.mark.parametrize("plan,cfg_name", [("P1", "c1mg"), ("P3", "c1mg"), ("P4", "c1mg"), ("P6", "c1mg"),
                                           ("P1", "c1g"), ("P6", "c1g")])
def test_gqa_multi_gpu_plans(plan, cfg_name, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
           str(out), "2", cfg_name]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    _ok(json.loads(out.read_text()))


@pytest.mark.parametrize("cfg_name", ["c1g", "c1mg"])
def test_gqa_p0_fp32(cfg_name):
    """FP32 parity mode with GQA (SIMT attention, any head_dim): <= 1e-4 against the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from tests.mp_worker import run
    from tests.test_gpu_fp32 import _assert_fp32
    _assert_fp32(run("P0", steps=2, cfg_name=cfg_name, dtype="fp32"))


@pytest.mark.parametrize("plan", ["P1", "P4"])
def test_gqa_multi_gpu_fp32(plan, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = WORLD[plan]
    if torch.cuda.device_count() < n:
        pytest.skip(f"{plan} needs {n} GPUs")
    from tests.test_gpu_fp32 import _assert_fp32
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29538", os.path.join(ROOT, "tests", "mp_worker.py"), plan,
           str(out), "2", "c1g", "fp32"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    _assert_fp32(json.loads(out.read_text()))


def test_gqa_plan_rejections():
    """A head split that cuts a KV group is refused at plan time (E_PLAN), not mid-step."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from synth.gen import C1_MED_GQA
    from paper_2410_13333_b200 import plans as Pl
    from paper_2410_13333_b200 import _lib as L
    from paper_2410_13333_b200.engine import Engine
    cfg = C1_MED_GQA
    ok = Pl.plan([Pl.pipe([Pl.stage([0], [4], [cfg.ffn], [cfg.vocab], [0, cfg.n_layers])], 4)], 2, 8)
    e = Engine(cfg, 0, 1, 0)
    e.apply(ok)
    e.close()
    bad = Pl.plan([Pl.pipe([Pl.stage([0, 1], [3, 1], [768, 768], [1024, 1024], [0, cfg.n_layers])], 4)], 2, 8)
    e = Engine(cfg, 0, 1, 0)
    with pytest.raises(L.MalleusError, match="KV groups"):
        e.requirements(bad)
    e.close()
