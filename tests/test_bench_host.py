"""Host logic of bench.py and the multi-process control plane, CPU only: workload resolution
per GPU count (headline + north-star extras), the reference arm printing the GPU arm's exact
config, the B1 pairing against the oracle's rank grid, and a world_size-2 gloo run of the
bootstrap (blob all-gather, ppc_connect, DCBS groups) with host-only comms."""
import json
import os
import socket

import pytest
import torch.multiprocessing as tmp

import bench
from oracle.groups import build_groups


def test_resolve_headline_and_extras():
    a = bench.parse([])
    w1 = bench.resolve(a, 1)
    assert (w1["virtual"], w1["pp"], w1["M"], w1["msg_bytes"], w1["chunk"], w1["slots"]) == \
        (True, 2, 8, 4096 * 4096 * 2, 128 << 10, 3)
    assert not w1["zc"]                                # no NVLink on one GPU
    for n, pipes in ((2, 1), (4, 2), (8, 4)):
        w = bench.resolve(a, n)
        assert (w["virtual"], w["pipelines"], w["dp"], w["zc"], w["chunk"]) == \
            (False, pipes, pipes, True, 256 << 10)
    c3, c4 = bench.resolve(a, 8, "C3"), bench.resolve(a, 8, "C4")
    assert (c3["pp"], c3["tp"], c3["M"], c3["pipelines"], c3["zc"]) == (4, 2, 16, 2, False)
    assert (c4["pp"], c4["M"], c4["msg_bytes"], c4["pipelines"]) == (8, 32, 4096 * 3584 * 2, 1)
    assert bench.EXTRA[4] == ["C3-pp4", "C4-pp4"] and bench.EXTRA[8] == ["C3", "C4"]
    with pytest.raises(SystemExit):
        bench.resolve(a, 1, "C3")                      # 8 ranks' worth on one GPU
    with pytest.raises(SystemExit):
        bench.resolve(a, 6, "C4")


def test_reference_arm_prints_the_gpu_arms_config(monkeypatch, capsys):
    monkeypatch.setattr(bench, "oracle_step", lambda pp, M, nb, seed=42: 0.01)
    monkeypatch.setattr(bench, "cpu_model", lambda: "test-cpu")
    for n in (1, 2, 8):
        a = bench.parse(["--impl", "reference", "--gpus", str(n), "--steps", "3", "--warmup", "1"])
        bench.run_reference(a)
        line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
        assert line["config"] == bench.config_dict(bench.resolve(a, n), n)
        assert line["impl"] == "reference" and line["n_gpus"] == n and line["steps"] == 3
        w = bench.resolve(a, n)
        assert line["value"] == pytest.approx(w["pipelines"] * w["M"] * w["seq"] / 0.01)
        for k in ("metric", "unit", "higher_is_better", "cpu_baseline", "e2e", "dtype", "data"):
            assert k in line
        assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.parametrize("world", [2, 4, 8])
def test_b1_pairs_follow_the_rank_grid(world):
    """Each B1 pair = the two stages of one PP pipeline of the oracle's DCBS grid."""
    g = build_groups(world, tp=1, pp=2, dp=world // 2)
    for r in range(world):
        st, lead = bench.b1_pair(r, world)
        pipe = next(p for p in g["pp"] if r in p)
        assert pipe.index(r) == st and pipe[0] == lead


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_18007_b200 as ppc
    cfg = ppc.make_config(tp=2, pp=world // 2, dp=1)
    comm = ppc.connect_distributed(cfg, rank, world, -1, with_nccl=False)   # host-only comm
    out = {g: comm.group(g) for g in (ppc.GROUP_TP, ppc.GROUP_DP, ppc.GROUP_PP)}
    t = [0.0]
    import torch
    v = torch.tensor([float(rank)])
    dist.all_reduce(v, op=dist.ReduceOp.MAX)             # bench's max-over-ranks reduction
    q.put((rank, {g: (m, b) for g, (m, b) in out.items()}, float(v.item())))
    comm.disconnect()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_bootstrap_world(world):
    """world_size-2 / 4 gloo processes on CPU: blob all-gather + ppc_connect of host-only
    comms, DCBS groups (TP / DP on NCCL, PP on the peer path) equal to the oracle's grid,
    and the max-over-ranks all-reduce bench.py times with."""
    import paper_2602_18007_b200 as ppc
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = build_groups(world, tp=2, pp=world // 2, dp=1)
    for rank, groups, vmax in res:
        assert vmax == world - 1
        tp_m, tp_b = groups[ppc.GROUP_TP]
        pp_m, pp_b = groups[ppc.GROUP_PP]
        assert tp_m == next(x for x in g["tp"] if rank in x) and tp_b == ppc.BACKEND_NCCL
        assert pp_m == next(x for x in g["pp"] if rank in x) and pp_b == ppc.BACKEND_PEER


def test_committed_ncu_counters_give_the_pull_protocol_bounds():
    """The NVLink counters behind roofline.protocol_bound (profiles/ncu_traffic.json): user
    bytes = one 32 MiB message; 16 B of response header per 128 B on rx, 24 B of request per
    128 B on tx — so 800 GB/s one way, 685.7 GB/s with both directions pulling."""
    nvl = bench.ncu_traffic("recv_n2_nvl_totals")
    assert nvl["user_bytes"] == 32 << 20
    assert nvl["nvlrx_bytes"] - nvl["user_bytes"] == pytest.approx(nvl["user_bytes"] * 16 / 128, rel=1e-5)
    assert nvl["nvltx_bytes"] == pytest.approx(nvl["user_bytes"] * 24 / 128, abs=128)   # + the credit
    assert 900 * nvl["user_bytes"] / nvl["nvlrx_bytes"] == pytest.approx(800.0, rel=1e-5)
    assert 900 * nvl["user_bytes"] / (nvl["nvlrx_bytes"] + nvl["nvltx_bytes"]) == pytest.approx(685.7, rel=1e-3)
