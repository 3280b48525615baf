"""Speed probe (CUDA-event timing, straggling rate = slowdown vs a normal GPU)
and straggler emulation (reading R13: the injected rate is calibrated until the
probe measures it within 5%)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from synth.gen import C1_TINY
    from paper_2410_13333_b200.engine import Engine
    e = Engine(C1_TINY, 0, 1, 0)
    yield e
    e.close()


def test_probe_uniform_repeatable(eng):
    a = eng.probe(10)[0]
    b = eng.probe(10)[0]
    assert a > 0 and abs(a / b - 1) < 0.05


def test_duty_slows_and_recovers(eng):
    t0 = eng.probe(10)[0]
    eng.set_slowdown(2.0, 2)
    t1 = eng.probe(10)[0]
    eng.set_slowdown(1.0, 0)
    t2 = eng.probe(10)[0]
    assert 1.4 < t1 / t0 < 3.0, (t0, t1)
    assert abs(t2 / t0 - 1) < 0.1, (t0, t2)


@pytest.mark.parametrize("x", [1.5, 2.0])
def test_calibration_hits_target(eng, x):
    nominal, measured = eng.calibrate_slowdown(0, x)
    eng.set_slowdown(1.0, 0)
    assert abs(measured / x - 1) <= 0.05, (nominal, measured)


def test_hog_mode_refused(eng):
    """HOG (a resident SM-occupying kernel) deadlocks device-wide syncs; the library refuses it."""
    from paper_2410_13333_b200 import _lib as L
    assert L.lib.malleus_set_slowdown(eng.ctx, 2.0, 1) == 1
