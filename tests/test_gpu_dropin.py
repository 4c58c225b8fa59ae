"""The C++ drop-in (include/rkfac_gpu.hpp) against the reference's own FP64 functions, same inputs and RngState,
through the reference's types (oracle/_ref/dropin_test, built from tests/cpp/dropin_test.cpp by oracle/Makefile)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in check not built (needs the reference headers)")
def test_cpp_dropin_matches_reference():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0, res
    assert res["fails"] == 0 and res["damping_throws"] == 1
    for m in ("srevd", "rsvd_psd"):
        assert res[m]["counter_match"] == 1
        assert res[m]["recon"] < 1e-4 and res[m]["eig"] < 1e-4 and res[m]["precond"] < 1e-4
    # the batched optimizer step (include/rkfac_gpu_optimizer.hpp) vs rkfac::optimizer_step on an identical net over
    # the T_KI cache schedule, SRE-KFAC and RS-KFAC: updates and the mirrored cached decompositions
    opt = res["optimizer_step"]
    assert opt["cache_ok"] == 1 and opt["updates"] < 1e-4 and opt["cached_recon"] < 1e-4
