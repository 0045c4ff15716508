"""Row-sharded mode (psdproj_create_sharded) with 2 and 3 ranks on ONE GPU: ranks are
host threads of one process and the collectives go through an in-process loopback NCCL
(tests/nccl_loopback.cu via PSDPROJ_NCCL_LIB; the pool provides one GPU). Exercises the per-rank row
offsets, pack/unpack of the all-gathered directions, the all-reduced Gram partials and column norms,
the replicated Rayleigh-Ritz (identical decisions on every rank) and Pi_local = W_local W^T. Checks:
the assembled Pi against O-EXACT (BJ threshold), against the unsharded context, exact symmetry,
every rank reporting identical info, and the bound dominating the error."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nccl_loopback.cu")
SO = os.path.join(HERE, "libnccl_loopback.so")


def _build():
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, SRC])
    return SO


@pytest.mark.parametrize("world,case", [(2, "c1"), (3, "c1"), (2, "odd_neg")])
def test_sharded_loopback(api, world, case):
    env = dict(os.environ, PSDPROJ_NCCL_LIB=_build())
    out = subprocess.run([sys.executable, os.path.join(HERE, "sharded_loopback_run.py"), str(world), case],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in res, res
    for row in res["rows"]:
        assert row["status"] in (0, 1), row
        assert row["rel_err_oracle"] <= 1e-9, row
        assert row["rel_diff_unsharded"] <= 1e-11, row
        assert row["err_bound"] >= row["err"], row
        assert row["symmetric"] and row["ranks_agree"], row
    if case == "odd_neg":
        assert any(r["side"] == -1 for r in res["rows"])
