"""Host logic of the C++ facade's multi-GPU trainer (include/vqmc_b200/vqmc.hpp, one host thread and
NCCL rank per GPU): which reference workers and streams each rank plays (trainer.cpp:121-127, 284-287)
must be the same partition as the Python data-parallel plan (paper_2106_13308_b200/dp.py) that the
gloo tests check against the oracle.  Compiled and run here (no GPU needed)."""
import os
import subprocess

import pytest

from paper_2106_13308_b200 import dp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#include <cstdio>
#include "vqmc_b200/vqmc.hpp"
int main() {
  const int cases[][2] = {{1, 1}, {4, 2}, {8, 8}, {6, 3}, {16, 4}};
  for (auto& c : cases) {
    vqmc::RunConfig cfg;
    cfg.workers = c[0];
    cfg.gpus = c[1];
    cfg.device = 1;
    for (int r = 0; r < cfg.gpus; ++r) {
      const auto p = vqmc::detail::rank_plan(cfg, r);
      std::printf("%d %d %d %d %d %llu\n", c[0], c[1], r, p.workers, p.device, (unsigned long long)p.stream0);
    }
  }
  vqmc::RunConfig bad;
  bad.workers = 3;
  bad.gpus = 2;
  try {
    vqmc::detail::rank_plan(bad, 0);
  } catch (const std::invalid_argument& e) {
    std::printf("error %s\n", e.what());
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def plan_lines(tmp_path_factory):
    d = tmp_path_factory.mktemp("facade")
    src = d / "plan.cpp"
    src.write_text(SRC)
    exe = d / "plan"
    lib = os.path.join(ROOT, "paper_2106_13308_b200", "lib")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", lib, "-lvqmc_b200", f"-Wl,-rpath,{lib}", "-lpthread"], check=True)
    return subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.strip().split("\n")


def test_rank_plan_matches_python_plan(plan_lines):
    rows = [list(map(int, ln.split())) for ln in plan_lines if not ln.startswith("error")]
    assert len(rows) == 1 + 2 + 8 + 3 + 4
    for L, G, r, wr, dev, s0 in rows:
        p = dp.RankPlan(r, G, L // G)
        assert wr == p.workers_per_rank and s0 == p.stream0 and dev == 1 + r
    # every reference worker is played exactly once, by consecutive streams 1..L
    for L, G in {(row[0], row[1]) for row in rows}:
        streams = sorted(s0 + s for (l_, g_, r, wr, dev, s0) in rows if (l_, g_) == (L, G) for s in range(wr))
        assert streams == list(range(1, L + 1))


def test_rank_plan_rejects_uneven_split(plan_lines):
    assert any(ln == "error workers must be a multiple of gpus" for ln in plan_lines)
