"""Clock sampling during timed regions and the measured peak numbers the
rooflines are reported against (bench.py and the EP bench)."""

from __future__ import annotations

import json
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def measured_peaks():
    """MEASURED_PEAKS.json (driver-written on this pool's B200s), else the
    profiling recipe's fallback numbers."""
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def fp4_peaks():
    """Dense NVFP4 peak measured on this B200 pool (MEASURED_PEAKS.json has no FP4
    entry): cuBLASLt block-scaled NVFP4 8192^3 (scripts/measure_fp4_peak.py ->
    profiles/r02/fp4_peak.json), burst and sustained, with the clocks they ran at.
    -> (burst TFLOP/s, sustained TFLOP/s, source)."""
    f = ROOT / "profiles" / "r02" / "fp4_peak.json"
    if f.exists():
        d = json.loads(f.read_text())["nvfp4"]
        return float(d["burst_tflops"]), float(d["sustained_tflops"]), "profiles/r02/fp4_peak.json (measured)"
    return 5950.0, 5950.0, "round-1 constant (scripts/bench_fp4.py)"


FP4_TFLOPS_MEASURED = fp4_peaks()[0]


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML polled
    every 2 ms from a background thread; nvidia-smi cannot start fast enough for
    a sub-second region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int = 0, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples, self.reason_bits, self.max_mhz = [], 0, None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.reason_bits |= nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        sm = sorted(self.samples)
        reasons = sorted(n for n, b in self.REASONS.items() if self.reason_bits & b)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "NVML, 2 ms polling"}
