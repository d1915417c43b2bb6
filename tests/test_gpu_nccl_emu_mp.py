"""GPU: the slab decomposition in its deployment shape -- one PROCESS per rank,
launched by torchrun -- with 2-3 ranks on one B200, through the multi-process NCCL
emulator (tests/nccl_emu/nccl_emu_mp.cu; real NCCL refuses two ranks on one GPU):
ghost planes by NCCL send/recv or by the fused kernel's peer stores over CUDA IPC,
all-reduced scalars, the REPLICA chain, broadcasts -- checked against the
single-domain context; and bench.py's multi-rank path (--gpus 2) end to end."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "nccl_emu", "libnccl_emu_mp.so")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun(nranks, args, env_extra=None, timeout=420):
    if not os.path.exists(LIB):
        pytest.skip("tests/nccl_emu/libnccl_emu_mp.so not built (__graft_entry__.build)")
    env = dict(os.environ, PETTO_NCCL_LIB=LIB, OMP_NUM_THREADS="1", **(env_extra or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(nranks),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    if r.returncode != 0:
        errs = [x for x in r.stderr.splitlines() if "Error" in x or "error" in x or "[rank" in x]
        pytest.fail("\n".join(errs[:40]) + "\n" + r.stdout[-2000:])
    return json.loads([x for x in r.stdout.strip().splitlines() if x.startswith("{")][-1])


CASES = [(2, "replica", "z", "nccl"), (3, "replica", "z", "nccl"), (2, "fast", "x", "peer"),
         (3, "fast", "x", "peer"), (3, "fast", "z", "peer"), (2, "fast", "x", "nccl")]


@pytest.mark.parametrize("nranks,mode,layout,halo", CASES)
def test_rank_processes_match_single_domain(nranks, mode, layout, halo):
    d = torchrun(nranks, [os.path.join(HERE, "nccl_emu", "run_ranks_mp.py"), mode, layout, halo])
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


@pytest.mark.parametrize("nranks,halo", [(2, "peer"), (2, "nccl"), (4, "peer")])
def test_bench_ranks(nranks, halo):
    """bench.py --gpus N as the driver launches it (torchrun, one process per rank):
    x-slabs, the halo, max-over-ranks timing, the e2e leg, one JSON line.  The
    ranks share one GPU here, so the numbers are not a scaling measurement."""
    d = torchrun(nranks, ["bench.py", "--gpus", str(nranks), "--config", "C4", "--steps", "3", "--warmup", "3",
                          "--no-cpu", "--halo", halo], {"PETTO_BENCH_DIST_BACKEND": "gloo"})
    print(d)
    assert d["n_gpus"] == nranks and d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["parallelism"].startswith(f"slab{nranks}")
    assert ("peer" in d["halo"]) == (halo == "peer")
