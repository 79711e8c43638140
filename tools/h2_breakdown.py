"""Where one H2 application goes, warm and graph-replayed (CUPTI via
torch.profiler, no kernel serialisation): per-kernel launches and time, the
sum of kernel durations against the elapsed time (the gap is launch / dependency
latency), and the launches per component level.

  python tools/h2_breakdown.py c2
"""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.composite import GpuCompositePreconditioner, gpu_composite_of  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
A = problems.CONFIGS[cfg]["build"]()
est = MultiVectorAMG().fit(A)
pc = GpuCompositePreconditioner(gpu_composite_of(est.composite_))
r = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
for _ in range(3):
    pc.apply_device(r)
torch.cuda.synchronize()
t0 = time.perf_counter()
pc.apply_device(r)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    pc.apply_device(r)
    torch.cuda.synchronize()
events = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
by = collections.defaultdict(lambda: [0, 0.0])
t_first, t_last, busy = None, None, 0.0
for e in events:
    name = e.name.split("(")[0]
    by[name][0] += 1
    by[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    s, d = e.time_range.start, e.time_range.end
    t_first = s if t_first is None else min(t_first, s)
    t_last = d if t_last is None else max(t_last, d)
total = sum(v[1] for v in by.values())
n = sum(v[0] for v in by.values())
print(f"{cfg}: components {est.composite_.n_components}, levels per component "
      f"{[c.operator.n_levels for c in est.composite_.components]}")
print(f"one application: wall {wall * 1e3:.1f} ms unprofiled; profiled span {(t_last - t_first) / 1e3:.1f} ms, "
      f"{n} kernels, sum of kernel durations {total / 1e3:.1f} ms ({100 * total / max(1, t_last - t_first):.0f}% "
      f"of the span), mean {total / max(1, n):.2f} us per kernel")
print(f"{'share':>7} {'launches':>9} {'mean us':>9}  kernel")
for name, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{100 * t / total:6.2f}% {c:9d} {t / c:9.2f}  {name[:90]}")
