"""Drive the NTT kernels on a large batch (microbench shape) for ncu / timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_18150_b200 import helrm  # noqa: E402

cfg = synth.config_by_name("criteo")
P = helrm.params_from_config(cfg)
stream = torch.cuda.Stream()
ctx = helrm.Context(P, 0, stream.cuda_stream)
limbs = int(sys.argv[1]) if len(sys.argv) > 1 else 64 * 48
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
buf = torch.randint(0, 2**49, (limbs * cfg.N,), dtype=torch.int64, device="cuda").view(torch.uint64)
torch.cuda.synchronize()
L = cfg.level + 1
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
helrm.ntt_fwd(ctx, buf, 0, L, limbs // L)
helrm.ntt_inv(ctx, buf, 0, L, limbs // L)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(reps):
    helrm.ntt_fwd(ctx, buf, 0, L, limbs // L)
e1.record(stream)
for _ in range(reps):
    helrm.ntt_inv(ctx, buf, 0, L, limbs // L)
e2.record(stream)
torch.cuda.synchronize()
f, i = e0.elapsed_time(e1) / reps, e1.elapsed_time(e2) / reps
gb = 16.0 * cfg.N * limbs / 1e9
bfly = limbs * cfg.N / 2 * 16
print(f"limbs {limbs}: fwd {f:.3f} ms {gb / f * 1e3:.0f} GB/s {bfly / f / 1e6:.0f} Gbfly/s | inv {i:.3f} ms {gb / i * 1e3:.0f} GB/s")
