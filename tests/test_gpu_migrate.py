"""Migration is bit-exact (BASELINE.json north star): params to new holders, fp32 master/m/v to new
owners, A -> B -> A round trip, received bytes == the oracle's delta bytes.  Multi-GPU (torchrun)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("pair,n", [("P2-P1", 2), ("P5-P6", 3), ("P4-swap", 4)])
def test_migration_bitexact(pair, n, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    out = tmp_path / "m.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "tests", "mp_migrate_worker.py"),
           pair, str(out)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, "\n".join(l for l in (p.stdout + p.stderr).splitlines()
                                        if "Error" in l or "error" in l or "rank" in l)[-6000:]
    r = json.load(open(out))
    assert r["ok"], r["errors"]
    assert r["bytes_recv"] == r["oracle_bytes"], r
