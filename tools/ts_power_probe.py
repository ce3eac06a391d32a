"""Power / clock of the phase-3 lmme_ts kernel (digest epilogue, batch 8192, d = 512) run back
to back for a few seconds, with nvidia-smi sampling power draw and SM clock. GOOM_TS_DEBUG
variants (profiling aids, wrong results): 1 = no TF32 split / plane stores in the transform,
2 = no MMA issue, 128 = constant operands. Shows which part of the kernel's energy the
1 kW power cap is paying for."""
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops  # noqa: E402

d, batch, secs = 512, 8192, float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
dev = torch.device("cuda")
L = ops.ts_random_normal(batch, d, 1, 0, dev)
C = ops.ts_random_normal(batch // 64, d, 2, 0, dev)
ops.lmme_ts(L, C, 2, b_div=64)
torch.cuda.synchronize()
rows = []
proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=power.draw,clocks.sm",
                         "--format=csv,noheader,nounits", "-lms", "100"],
                        stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l) for l in proc.stdout], daemon=True).start()
time.sleep(0.5)
n0 = len(rows)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t_end = time.time() + secs
reps = 0
a.record()
while time.time() < t_end:
    for _ in range(4):
        ops.lmme_ts(L, C, 2, b_div=64)
    reps += 4
    torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
rows_run = rows[n0:]
proc.terminate()
pw = [float(r.split(",")[0]) for r in rows_run if r.strip()]
mhz = [float(r.split(",")[1]) for r in rows_run if r.strip()]
ms = a.elapsed_time(b) / reps
print(f"debug={os.environ.get('GOOM_TS_DEBUG', '0')}: {ms:.2f} ms/launch "
      f"{2 * d**3 * batch / ms / 1e9:.0f} TF/s  power median {statistics.median(pw):.0f} W  "
      f"sm clock median {statistics.median(mhz):.0f} MHz  ({len(pw)} samples)", flush=True)
