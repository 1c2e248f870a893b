import os, sys, torch
sys.path.insert(0, "/root/repo")
os.environ["PPC_DEBUG"] = "1"
os.environ["PPC_LOCAL_DIRECT"] = "0"
import paper_2602_18007_b200 as ppc
S, M, n = 2, 4, 2 * (64 << 10) + 321
cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10)
comms = ppc.virtual_stages(cfg, 0)
X = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
G = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
Y = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
DX = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
for variant in ["identity", "xor"]:
    if variant == "xor":
        ctx = [(ppc.XorCtx(42, 0, s, 0), ppc.XorCtx(42, 0, s, 1)) for s in range(S)]
        args = [ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR, bwd=ppc.STAGE_XOR, fwd_user=ctx[s][0], bwd_user=ctx[s][1],
                             x=X if s == 0 else None, g=G if s == S - 1 else None, y=Y if s == S - 1 else None, dx=DX if s == 0 else None) for s in range(S)]
    else:
        args = [ppc.StepArgs(M, n, n, x=X if s == 0 else None, g=G if s == S - 1 else None, y=Y if s == S - 1 else None, dx=DX if s == 0 else None) for s in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    ppc.step_1f1b_local(comms, args, streams)
    torch.cuda.synchronize()
    try:
        g = ppc.StepGraph(comms, args, streams)
        g.launch(); torch.cuda.synchronize(); print(variant, "graph OK", flush=True)
    except Exception as e:
        print(variant, "graph FAILED", e, flush=True)
