"""Run the in-run FP64 roofline probes once each (for ncu evidence)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_16877_b200 import abi
t = C.c_double()
assert abi.lib().hpac_probe_fp64_peak(C.byref(t)) == 0
print(f"fp64 DFMA probe {t.value:.2f} TFLOP/s")
assert abi.lib().hpac_probe_dmma_peak(C.byref(t)) == 0
print(f"DMMA m8n8k4 probe {t.value:.2f} TFLOP/s")
