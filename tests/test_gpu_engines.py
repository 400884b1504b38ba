"""Engine alternatives that the default routing does not pick for the test shapes, run in a
subprocess with the switch that forces them, against the same reference checks:
  TTG_TALL_ENGINE=persist  the persistent blocked in-place QRCP (DMMA panel updates; the default
                           only for square in-place problems >= 2048)
  TTG_TALL_ENGINE=steps    the per-step in-place kernels everywhere
  TTG_LAZY=0               plain per-step streams instead of candidate pivoting (narrow W)
  TTG_LZ_TAILS=0           the candidate engine's threshold / final choice / next first choice as
                           launches of their own instead of last-CTA tails of their predecessors
  TTG_LAZY_WIDE=0          the subspace engine instead of candidate pivoting on 32 < k <= 1024 (it is
                           the default only for 1024 < k <= 2048)
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(env_extra, select):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu", *select],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_persistent_inplace_engine():
    _run({"TTG_TALL_ENGINE": "persist"},
         ["tests/test_gpu_sweeps.py", "-k", "qr_col_pivot or general_paths or planted"])


def test_per_step_inplace_engine():
    _run({"TTG_TALL_ENGINE": "steps"}, ["tests/test_gpu_sweeps.py", "-k", "qr_col_pivot"])


def test_plain_streams_without_candidate_pivoting():
    _run({"TTG_LAZY": "0"}, ["tests/test_gpu_lazy.py", "-k", "planted"])


def test_subspace_engine_on_wide_cuts():
    _run({"TTG_LAZY_WIDE": "0"}, ["tests/test_gpu_lazy.py", "-k", "wide_second_cut"])


def test_candidate_engine_without_last_cta_tails():
    _run({"TTG_LZ_TAILS": "0"}, ["tests/test_gpu_lazy.py", "-k", "planted or wide_second_cut"])
