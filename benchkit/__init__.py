"""Bench infrastructure: peaks, clock sampling, FFMA probe, roofline arithmetic.

Not on the beamforming path.  Roofline per SURVEY.md §8(d) / DESIGN.md §Roofline:
  per block  FLOPs = 8 * n_ant * b * f          (30,720 f at n_ant=64, b=60)
             bytes = 8 * b * (f + n_ant)         (S read + R write; 480 (f + 64))
  P_FP32 = SMs x 128 FP32 lanes x 2 FLOP x clock  (derived from the guide's unit counts)
  HBM    = MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)
"""
from __future__ import annotations

import ctypes
import json
import os
import statistics
import subprocess
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbfprobe.so")

FP32_LANES_PER_SM = 128          # B200 SM: 4 SMSPs x 32 FP32 lanes
FLOP_PER_FMA = 2
FALLBACK = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    except (OSError, ValueError):
        return dict(FALLBACK)


def fp32_peak_tflops(sms: int, mhz: float) -> float:
    return sms * FP32_LANES_PER_SM * FLOP_PER_FMA * mhz * 1e6 / 1e12


def ffma_probe(iters: int = 4096, ctas_per_sm: int = 4) -> dict:
    """Measured FFMA throughput of every SM (3-register FFMA outer product)."""
    L = ctypes.CDLL(LIB_PATH)
    L.bfp_ffma_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    L.bfp_ffma_peak.restype = ctypes.c_int
    tf, ms, sms = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    rc = L.bfp_ffma_peak(iters, ctas_per_sm, ctypes.byref(tf), ctypes.byref(ms), ctypes.byref(sms))
    if rc:
        raise RuntimeError(f"bfp_ffma_peak failed ({rc})")
    return {"tflops": tf.value, "ms": ms.value, "sms": sms.value}


class ClockSampler:
    """nvidia-smi sampling of SM clock, power and throttle reasons during a timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "utilization.gpu")

    def __init__(self, gpu_index: int = 0, period_ms: int = 100):
        self.gpu, self.period = gpu_index, period_ms
        self.rows: list[list[str]] = []
        self._proc = None
        self._thread = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", f"-lms={self.period}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return self
        self._thread = threading.Thread(target=self._read, daemon=True)
        self._thread.start()
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self._proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self._proc.terminate()
        try:
            self._proc.wait(timeout=5)
        except subprocess.TimeoutExpired:  # pragma: no cover
            self._proc.kill()
        if self._thread:
            self._thread.join(timeout=5)
        return self.summary()

    def summary(self) -> dict:
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        load = [r for r in self.rows if (num(r[8]) or 0) > 50] or self.rows
        sm = [num(r[0]) for r in load if num(r[0]) is not None]
        mx = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[4 + i] == "Active"})
        pw = [num(r[2]) for r in load if num(r[2]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons,
                "power_w_max": max(pw) if pw else None,
                "power_w_median": statistics.median(pw) if pw else None,
                "samples": len(self.rows), "samples_under_load": len(load)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
