"""On-device C_peak calibration (Alg. 2; reference `sgrpo profile --real`, tools/sgrpo.cpp:30-66):
measure the batched-forward latency curve of a workload's target shape on this GPU, find the
knee (roofline.cpp:39-108) and write the reference's HardwareProfile JSON
(roofline.cpp:188-201) to profiles/hw_profile_<config>.json.

    python scripts/calibrate_cpeak.py [config] [b_max]
"""
import json
import os
import sys

sys.path.insert(0, '.')
from bench import WORKLOADS, measured_peaks, model_cfg  # noqa: E402
from paper_2509_21792_b200 import capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
b_max = int(sys.argv[2]) if len(sys.argv) > 2 else 512
w = dict(WORKLOADS[name])
eng = capi.Engine(model_cfg(w), 1, 0, 8, max(2048, b_max), 10, 6)
eng.init_random(1234)
r = eng.measure_c_peak(b_max, warmup=1, reps=5)
hbm, tf, _ = measured_peaks()
prof = {"name": f"B200 ({name} target shape, measured)", "peak_flops": tf * 1e12, "bandwidth": hbm * 1e9,
        "bytes_per_element": 2, "c_peak": r["c_peak"], "confidence": r["confidence"],
        "low_confidence": r["low_confidence"], "latency_curve": r["latency_curve"]}
os.makedirs("profiles", exist_ok=True)
out = f"profiles/hw_profile_{name}.json"
json.dump(prof, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in prof.items() if k != "latency_curve"}))
print("curve (b, ms):", [(b, round(s * 1e3, 3)) for b, s in r["latency_curve"][::max(1, b_max // 32)]])
