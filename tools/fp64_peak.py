"""Runs tools/fp64_peak.cu (burst + 4 s sustained) under the nvidia-smi clock sampler of bench.py and
writes profiles/fp64_peak.json with the clocks and throttle reasons seen during the run (GPU box)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402

exe = "/tmp/fp64_peak"
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                os.path.join(ROOT, "tools", "fp64_peak.cu")], check=True)
with ClockSampler(0) as clk:
    out = subprocess.run([exe, "4"], capture_output=True, text=True, check=True).stdout
d = json.loads(out)
d["clocks"] = clk.summary()
d["nominal_fp64_tflops"] = 37.2  # HGX B200 datasheet (non-tensor FP64), for the frac beside the measured one
with open(os.path.join(ROOT, "profiles", "fp64_peak.json"), "w") as f:
    json.dump(d, f, indent=1)
print(json.dumps(d))
