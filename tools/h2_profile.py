"""One H2 application (symmetrized composite of the bootstrap K-cycles) of a
fitted config between cudaProfilerStart/Stop, for an ncu launch list:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
      python tools/h2_profile.py c1
"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.composite import GpuCompositePreconditioner, gpu_composite_of  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
A = problems.CONFIGS[cfg]["build"]()
est = MultiVectorAMG().fit(A)
pc = GpuCompositePreconditioner(gpu_composite_of(est.composite_))
r = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
for _ in range(2):
    pc.apply_device(r)
torch.cuda.synchronize()
torch.cuda.profiler.start()
pc.apply_device(r)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("components", est.composite_.n_components, "levels",
      [c.operator.n_levels for c in est.composite_.components])
