import time, numpy as np, torch
x = np.random.rand(302 * 1024 * 1024 // 8)
d = torch.empty(x.size, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); d.copy_(torch.from_numpy(x)); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"pageable H2D {x.nbytes/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
p = torch.empty(x.size, dtype=torch.float64, pin_memory=True)
t0 = time.perf_counter(); p.numpy()[:] = x; dt = time.perf_counter() - t0
print(f"host memcpy into pinned {x.nbytes/dt/1e9:.1f} GB/s")
for rep in range(2):
    t0 = time.perf_counter(); d.copy_(p, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"pinned H2D {x.nbytes/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
import os; print("cpus", len(os.sched_getaffinity(0)))
