"""GPU: the NCCL branches of the slab decomposition with 2-4 ranks on one B200,
through the in-process NCCL emulator (tests/nccl_emu/nccl_emu.cu; real NCCL refuses
two ranks on one GPU).  Each rank is a host thread with its own slab context and
communicator -- one process per GPU's code path: ghost planes by send/recv every
step, all-reduced scalars, the REPLICA chain (send/recv + broadcast), node 0's
Lame pair broadcast -- checked against the single-domain context."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "nccl_emu", "libnccl_emu.so")


CASES = [(2, "replica", "z"), (3, "replica", "z"), (4, "replica", "z"), (2, "fast", "z"), (3, "fast", "z"),
         (2, "fast", "x"), (3, "fast", "x")]


@pytest.mark.parametrize("nranks,mode,layout", CASES)
def test_nccl_ranks_match_single_domain(nranks, mode, layout):
    if not os.path.exists(LIB):
        pytest.skip("tests/nccl_emu/libnccl_emu.so not built (__graft_entry__.build)")
    # eager module loading: a lazy kernel load may synchronise the device while a
    # rank's stream waits on an operation another rank thread has yet to post; one
    # hardware work queue per stream: a stream waiting on a flag blocks its queue
    env = dict(os.environ, PETTO_NCCL_LIB=LIB, CUDA_MODULE_LOADING="EAGER", CUDA_DEVICE_MAX_CONNECTIONS="32")
    r = subprocess.run([sys.executable, os.path.join(HERE, "nccl_emu", "run_ranks.py"), str(nranks), mode, layout],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print(d)
    assert d["ok"] and d["records_same_on_all_ranks"] and d["loops"][0] == d["loops"][1]
    assert d["state_bit_identical"]  # the state solve does not depend on the split
    assert abs(d["iters"][0] - d["iters"][1]) <= 1
    if mode == "replica":
        assert d["r_pde"][0] == d["r_pde"][1]
        assert d["records_bit_identical"] and d["phases_max_abs"] == 0.0
    else:
        assert abs(d["r_pde"][0] - d["r_pde"][1]) <= 1e-13 * d["r_pde"][1]
        assert d["records_max_rel"] <= 1e-12 and d["phases_max_abs"] <= 1e-12
