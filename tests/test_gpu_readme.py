"""The README quick start runs as written (at a smaller scale)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_readme_quickstart():
    import paper_2512_00705_b200 as dw
    g = dw.DeviceGraph.rmat(12, 16, seed=1)
    m = dw.Model("node2vec", a=0.5, b=2.0)
    ratio = dw.profile_edge_cost_ratio(g, m)
    assert ratio > 0
    opts = dw.RunOptions(walk_length=80, seed=7, edge_cost_ratio=ratio)
    res = dw.run_queries(g, m, np.arange(1 << 12, dtype=np.uint32), opts)
    assert res.stats["steps"] > 0
    p = res.paths[0][:res.lengths[0]]
    assert p[0] == 0 and len(p) == res.lengths[0]
