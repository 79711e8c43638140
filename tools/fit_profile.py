"""cProfile of MultiVectorAMG().fit on a config (where the setup time goes)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
A = problems.CONFIGS[name]["build"]()
MultiVectorAMG().fit(problems.CONFIGS["c1"]["build"]())  # warm-up (library load, allocator)
pr = cProfile.Profile()
pr.enable()
MultiVectorAMG().fit(A)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
