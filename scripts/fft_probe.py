"""cuFFT (torch.fft) throughput for the phi-stage row lengths: batched
complex128 FFTs of length n over `rows` rows, event-timed."""
import json
import sys

import torch

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
res = {}
for n in (4095, 8190, 8191, 16382, 16383):
    x = torch.randn((rows, n), dtype=torch.complex128, device="cuda")
    for _ in range(2):
        y = torch.fft.fft(x, dim=-1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        y = torch.fft.fft(x, dim=-1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    res[n] = {"ms": ms, "GBps_one_pass": 2 * x.numel() * 16 / (ms * 1e-3) / 1e9}
    del x, y
    torch.cuda.empty_cache()
print(json.dumps({"rows": rows, "fft": res}))
