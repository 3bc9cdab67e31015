import sys, os
sys.path.insert(0, '.')
from tests.test_gpu_fused_small import _simple, _treernn
from tests.helpers import gpu_ctx
for name, f, B in (("simple", _simple, 3), ("treernn", _treernn, 1)):
    dy, cg, m = gpu_ctx(seed=4, mb=64)
    w, l = f(dy, cg, m, B, False)
    c0 = cg._counters()[5]
    cg.forward_to(l)
    c1 = cg._counters()[5]
    print(name, os.environ.get("DG_AFFCELL", "1"), "forward launches", c1 - c0)
