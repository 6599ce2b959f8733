"""Host-side logic of bench.py that decides what the JSON line claims: the
tensor peak picked from the SM clock measured inside the FFN launches, and
that clock's estimate from the GEMM profile counters (CPU only)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

PEAKS = {"bf16_tflops": 1679.4, "bf16_tflops_sustained": 1426.3, "sm_max_mhz": 1965.0}


def test_peak_follows_the_in_kernel_clock():
    # kernels at max clock: burst; power-capped kernels: sustained, whatever NVML says
    t, src = bench.tensor_peak(PEAKS, {"sm_mhz": 1965.0, "sm_max_mhz": 1965}, 1950.0)
    assert t == 1679.4 and "burst" in src
    t, src = bench.tensor_peak(PEAKS, {"sm_mhz": 1965.0, "sm_max_mhz": 1965}, 1500.0)
    assert t == 1426.3 and "sustained" in src and "1500 MHz" in src
    # no in-kernel clock: the NVML sample decides
    assert bench.tensor_peak(PEAKS, {"sm_mhz": 1965.0, "sm_max_mhz": 1965})[0] == 1679.4
    assert bench.tensor_peak(PEAKS, {"sm_mhz": 1400.0, "sm_max_mhz": 1965})[0] == 1426.3
    assert bench.tensor_peak(PEAKS, None)[0] == 1679.4


class _FakeLib:
    """sida_debug_gemm_prof stand-in: per CTA, epilogue cycles in slot 5 and
    %globaltimer ns past the PDL wait (9) and at exit (10)."""

    def __init__(self, mhz, status=0):
        self.mhz, self.status = mhz, status

    def sida_debug_gemm_prof(self, ptr):
        if self.status:
            return self.status
        buf = np.ctypeslib.as_array(
            (np.ctypeslib.ctypes.c_uint64 * (2 * 148 * 12)).from_address(ptr)).reshape(2, 148, 12)
        span_ns = 200_000
        for g in range(2):
            buf[g, :, 9] = 1_000_000
            buf[g, :, 10] = 1_000_000 + span_ns
            buf[g, :, 5] = int(span_ns * self.mhz[g] / 1e3)
        return 0


def test_kernel_clock_from_profile_counters():
    mhz = bench.ffn_kernel_clock_mhz(_FakeLib((1400.0, 1600.0)))
    assert abs(mhz - 1500.0) < 1.0
    assert bench.ffn_kernel_clock_mhz(_FakeLib((1400.0, 1600.0), status=5)) is None
