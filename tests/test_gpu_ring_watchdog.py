"""The ring watchdog (flag-progress watchdog): a device wait on a
ready / credit word nobody will ever publish gives up after the timeout
instead of hanging the GPU, records the stall once, and the record re-arms."""
import ctypes as C
import time

import pytest
import torch

from paper_2411_12780_b200 import _native as N

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def test_ring_wait_times_out_and_reports():
    lib = N.load()
    words = torch.zeros(4, dtype=torch.int32, device="cuda")
    st = C.c_int * 4
    out = st()
    lib.ppll_ring_stall(out, 1)                      # clear any earlier record
    s = torch.cuda.current_stream().cuda_stream
    try:
        lib.ppll_set_ring_timeout_ms(50)
        N.check(lib.ppll_ring_publish(words.data_ptr(), 3, s), "publish")
        N.check(lib.ppll_ring_wait(words.data_ptr(), 3, s), "wait ok")      # already published
        torch.cuda.synchronize()
        assert lib.ppll_ring_stall(out, 0) == 0
        t0 = time.perf_counter()
        N.check(lib.ppll_ring_wait(words.data_ptr(), 7, s), "wait")          # never published
        N.check(lib.ppll_ring_wait_credit(words.data_ptr() + 4, 2, s), "credit")
        torch.cuda.synchronize()
        assert time.perf_counter() - t0 < 5.0
        assert lib.ppll_ring_stall(out, 1) == 1
        assert list(out) == [1, 7, 3, 0]                # first stall: the ready flag
        assert lib.ppll_ring_stall(out, 0) == 0         # re-armed
    finally:
        lib.ppll_set_ring_timeout_ms(30000)
