"""CPU checks of the C-ABI library: it loads, exports every entry point declared in
include/vqmc_b200.h, and its host utilities (no GPU needed) agree with the oracle."""
import os
import re

import numpy as np
import pytest

import pyoracle as O
from paper_2106_13308_b200 import _capi as K
from paper_2106_13308_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vqmc_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vqmc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    declared = _declared()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(K.lib, name), name
    assert sorted(K.EXPORTS) == declared


def test_made_init_matches_oracle_bitwise():
    for n, h, seed in ((4, 5, 0), (20, 45, 3), (100, 106, 7)):
        m = api.made_init(n, h, seed)
        o = O.made_init(n, h, seed)
        assert np.array_equal(m.degrees, o.degrees)
        assert np.array_equal(m.parameters(), o.theta)
    assert [api.default_made_hidden(n) for n in (4, 12, 20, 10000)] == [10, 31, 45, 424]
    with pytest.raises(ValueError):
        api.made_init(1, 4, 0)


def test_graphs_match_oracle():
    for n, s in ((20, 0), (100, 2)):
        assert np.array_equal(api.random_maxcut_graph(n, s).edges, O.random_maxcut_graph(n, s))
    assert np.array_equal(api.random_regular_graph(1000, 3, 4).edges, O.random_regular_graph(1000, 3, 4))
    assert np.array_equal(api.erdos_renyi_graph(50, 0.3, 1).edges, O.erdos_renyi_graph(50, 0.3, 1))


def test_stream_uniforms_match_oracle():
    s = api.make_stream(5, 7)
    a = s.uniforms(100)
    b = s.uniforms(50)
    ref = O.uniforms(5, 7, 150)
    assert np.array_equal(np.concatenate([a, b]), ref)
    assert api.mix_seed(3, 9) == O.mix_seed(3, 9)


def test_graph_io_roundtrip(tmp_path):
    g = api.random_maxcut_graph(8, 2)
    p = str(tmp_path / "g.txt")
    api.save_graph(g, p)
    h = api.load_graph(p)
    assert h.n == 8 and np.array_equal(h.edges, g.edges)
    for bad in ("graph 3\nedge 1 4\n", "graph 3\nedge 2 2\n", "graph 3\nedge 1 2\nedge 2 1\n", "tim 3\n"):
        (tmp_path / "b.txt").write_text(bad)
        with pytest.raises(RuntimeError):
            api.load_graph(str(tmp_path / "b.txt"))
    (tmp_path / "c.txt").write_text("# comment\ngraph 2 # two\nedge 1 2\n")
    assert api.load_graph(str(tmp_path / "c.txt")).edges.tolist() == [[0, 1]]


def test_maxcut_spec_validates():
    with pytest.raises(ValueError):
        api.maxcut_spec(api.Graph(3, np.array([[1, 0]])))
    with pytest.raises(ValueError):
        api.maxcut_spec(api.Graph(3, np.array([[0, 1], [0, 1]])))
    assert api.maxcut_spec(api.Graph(3, np.array([[0, 1], [1, 2]]))).num_edges == 2


def test_pooled_stats_exact():
    import ctypes as C
    rng = np.random.default_rng(0)
    E = 150
    cuts = rng.integers(60, 100, size=1024)
    l = 0.25 * (E - 2.0 * cuts)
    m, v = C.c_double(), C.c_double()
    K.check(K.lib.vqmc_pooled_stats(E, len(cuts), int(cuts.sum()), int((cuts ** 2).sum()), C.byref(m), C.byref(v)))
    rm, rv = O.energy_and_variance(l)
    assert m.value == rm and v.value == rv


def test_bit_packing_roundtrip():
    x = np.random.default_rng(1).integers(0, 2, (7, 100)).astype(np.uint8)
    w = K.pack_bits(x)
    assert w.shape == (7, 4) and np.array_equal(K.unpack_bits(w, 100), x)
    assert int(w[2, 1]) == sum(int(x[2, 32 + i]) << i for i in range(32))
