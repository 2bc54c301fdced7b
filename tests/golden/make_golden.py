"""Generates the committed golden fixtures from the CPU oracle (which is pinned to the
reference's own recorded outputs, tests/test_oracle_pins.py).  The reference itself cannot
be built here (Eigen3 / vendor/ absent), so these are oracle outputs.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as O  # noqa: E402


def make(n, B, seed, graph="maxcut"):
    h = O.default_made_hidden(n)
    m = O.made_init(n, h, seed)
    m.theta = m.theta + (O.uniforms(seed, 98, m.d) * 3.0 + -1.5)  # acceptance.cpp:87-92 perturbation
    edges = O.random_maxcut_graph(n, seed) if graph == "maxcut" else O.random_regular_graph(n, 3, seed)
    U = O.uniforms(seed, 1, n * B).reshape(n, B)  # worker 0's stream make_stream(seed, 1)
    x, lp, p = O.auto_sample(m, B, uniforms=U, want_p=True)
    le, cut = O.local_energy(n, edges, x)
    grad = O.gradient_from_locals(m, x, le)
    np.savez_compressed(os.path.join(HERE, f"oracle_n{n}_seed{seed}.npz"), n=n, h=h, B=B, degrees=m.degrees,
                        theta=m.theta, edges=edges, uniforms=U, x=x, log_psi=lp, p=p, cut=cut, local=le, grad=grad)


if __name__ == "__main__":
    make(20, 64, 0)
    make(100, 32, 1, graph="regular")
