"""Cross-process parity: one process per rank (torchrun), CUDA-IPC-mapped rings, device-side
flags/credits, over NVLink when each rank has its own GPU.  With fewer GPUs than ranks the
ranks share GPUs (time-sliced), so the whole cross-process protocol also runs on one GPU;
only the NCCL cases that need a GPU per rank are skipped then."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

HERE = os.path.dirname(os.path.abspath(__file__))
PORT = [29611]


# cases that need one GPU per rank: NCCL refuses two ranks of a communicator on one GPU
NEEDS_OWN_GPU = {("dcbs", 4), ("hetero", 4)}


# Every (case, ranks, env) of this file.  The cases of one rank count run in ONE torchrun
# session (mp_worker --batch: same checks, each case with its own comms and environment),
# which saves a process-group start-up per case; a case the batch did not report OK is run
# again on its own, so a batch failure can never hide or fake a result.
PLAN = [(c, 2, {}) for c in ("sendrecv_sm", "sendrecv_ce", "sendrecv_pull", "xor_sm", "xor_ce",
                             "xor_pull", "timeout", "toy", "inplace", "xor_inplace", "hetero",
                             "zc", "zc_unfused", "zc_side", "zc_bidir_stream", "zc_async",
                             "host", "graph", "fullsize")] + \
       [(c, 2, {"PPC_RECV_EARLY": "1"}) for c in ("zc", "zc_bidir_stream", "zc_async", "graph")] + \
       [(c, 2, {"PPC_STEP_BATCH": "1"}) for c in ("zc", "graph")] + \
       [("dcbs1", 2, {"PPC_NCCL_SINGLETON": "1"}), ("dcbs1", 3, {"PPC_NCCL_SINGLETON": "1"})] + \
       [(c, 4, {}) for c in ("inplace", "xor_inplace", "xor_sm", "xor_ce", "xor_pull", "hetero",
                             "host", "graph", "fullsize", "gather", "dcbs")]
_BATCH = {}


def _torchrun(n, args, timeout, env=None):
    PORT[0] += 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(PORT[0]),
           os.path.join(HERE, "mp_worker.py"), *args]
    try:
        return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                              env=None if env is None else {**os.environ, **env})
    except subprocess.TimeoutExpired as e:
        return subprocess.CompletedProcess(cmd, -1, e.stdout or "", e.stderr or "")


def _batch(n):
    """Run every planned case with n ranks in one torchrun session (once per module)."""
    if n not in _BATCH:
        plan = [(c, e) for c, k, e in PLAN if k == n and not
                (torch.cuda.device_count() < n and (c, n) in NEEDS_OWN_GPU)]
        r = _torchrun(n, ["--batch", json.dumps(plan)], timeout=120 + 40 * len(plan))
        out = r.stdout if isinstance(r.stdout, str) else r.stdout.decode(errors="replace")
        _BATCH[n] = {(c, json.dumps(e, sort_keys=True)): out.count(f"#{i} {c} OK") == n
                     for i, (c, e) in enumerate(plan)}
    return _BATCH[n]


def _run(case, n, timeout=240, env=None):
    """torchrun n ranks of tests/mp_worker.py.  With fewer GPUs than ranks the ranks share
    the GPUs round-robin (mp_worker.dev): still one process per rank, CUDA-IPC-mapped rings,
    device flag / credit / header spins — the GPU time-slices the processes."""
    if torch.cuda.device_count() < n and (case, n) in NEEDS_OWN_GPU:
        pytest.skip(f"needs {n} GPUs (NCCL: one GPU per rank)")
    key = (case, json.dumps(env or {}, sort_keys=True))
    if os.environ.get("PPC_TEST_NO_BATCH") != "1" and _batch(n).get(key):
        return                                   # passed inside the batch session
    r = _torchrun(n, [case], timeout, env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(f"{case} OK") == n


@pytest.mark.parametrize("case", ["sendrecv_sm", "sendrecv_ce", "sendrecv_pull", "xor_sm", "xor_ce", "xor_pull",
                                  "timeout", "toy"])
def test_two_gpus(case):
    _run(case, 2)


@pytest.mark.parametrize("n", [2, 4])
def test_produce_in_place_chain(n):
    _run("inplace", n)


@pytest.mark.parametrize("n", [2, 4])
def test_step_produce_in_place(n):
    _run("xor_inplace", n)


@pytest.mark.parametrize("case", ["xor_sm", "xor_ce", "xor_pull"])
def test_four_gpu_pipeline(case):
    _run(case, 4)


def test_dcbs_pp2_tp2():
    _run("dcbs", 4)


@pytest.mark.parametrize("n", [2, 3])
def test_dcbs_nccl_singleton_groups(n):
    """DCBS group init with NCCL communicators that any box can build (one-rank TP / DP
    groups; the ranks may share one GPU): NCCL init + allreduce through the C ABI beside a
    PP step, PP collectives refused."""
    _run("dcbs1", n, env={"PPC_NCCL_SINGLETON": "1"})


@pytest.mark.parametrize("n", [2, 4])
def test_hetero_allreduce(n):
    _run("hetero", n)


@pytest.mark.parametrize("case", ["zc", "zc_unfused", "zc_side"])
def test_zero_copy_registered_pull(case):
    """Default: the step driver fuses each source op's publication into the preceding
    terminal receive kernel; the other two cases cover the unfused publication kernel on
    the compute stream and on the send stream."""
    _run(case, 2)


def test_zero_copy_bidirectional_stream():
    _run("zc_bidir_stream", 2)


@pytest.mark.parametrize("case", ["zc", "zc_bidir_stream", "zc_async", "graph"])
def test_zero_copy_early_receive(case):
    """PPC_RECV_EARLY=1: receives look for their publication before griddepcontrol.wait
    and pull their first 64 KiB early (a stale graph sequence base must be discarded)."""
    _run(case, 2, env={"PPC_RECV_EARLY": "1"})


def test_zero_copy_async_sends():
    _run("zc_async", 2)


@pytest.mark.parametrize("n", [2, 4])
def test_step_with_host_buffers(n):
    _run("host", n)


@pytest.mark.parametrize("n", [2, 4])
def test_step_cuda_graph(n):
    _run("graph", n)


@pytest.mark.parametrize("n", [2, 4])
def test_full_size_bench_configuration(n):
    """C2 (2 GPUs) / C4 stand-in (4 GPUs) at full size in bench.py's launch configuration."""
    _run("fullsize", n, timeout=600)


def test_tp_sliced_boundary_fused_gather():
    """NEXT-1 on 4 GPUs (PP=2 x TP=2)."""
    _run("gather", 4)


@pytest.mark.parametrize("case", ["zc", "graph"])
def test_step_batched_terminal_receives(case):
    """PPC_STEP_BATCH=1: each rank's terminal receives (and their fused publications) run as
    one batched-receive grid per step, eager and inside the step's CUDA graph."""
    _run(case, 2, env={"PPC_STEP_BATCH": "1"})
