"""K4/K5 MoE dispatch/combine across W instances on one GPU vs the CPU oracle.

Parity is unpinned by the reference (it has no MoE code); the oracle is our
restatement dcpora_moe_layer_f64: out_t = sum over top-k experts, ascending id,
of w * W_down(silu(W_gate x) * W_up x), fp64 over bf16 inputs.  Tolerance bf16
rel-L2 <= 2e-2 per token (north_star).
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("W,E,k,H,I,m_max", [
    (4, 8, 2, 256, 64, 64), (2, 16, 4, 512, 128, 64), (8, 32, 8, 256, 32, 64),
    # the exchange at cfg4 / cfg5 widths (Qwen3-30B-A3B: hidden 2048, 128 experts top-8;
    # DeepSeek-V3: hidden 7168, 256 experts top-8), narrow experts to keep the fp64 oracle short
    (8, 128, 8, 2048, 16, 16), (8, 256, 8, 7168, 16, 8)])
def test_dispatch_combine_matches_oracle(W, E, k, H, I, m_max):
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.moe import MoeInstance
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(W * 100 + E)
    inst = [MoeInstance(ctx, W, s, H, k, E, m_max) for s in range(W)]
    for s in range(W):
        for t in range(W):
            inst[s].set_peer_local(t, inst[t])
        inst[s].commit()
    w_gate = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_up = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_down = (torch.randn(E, H, I, generator=g, device=dev) / I ** 0.5).to(torch.bfloat16)
    toks = []
    for s in range(W):
        M = int(torch.randint(1, m_max + 1, (1,), generator=g, device=dev).item()) if s != 1 else 0
        x = torch.randn(M, H, generator=g, device=dev).to(torch.bfloat16)
        logits = torch.randn(M, E, generator=g, device=dev)
        top = torch.topk(logits, k, dim=-1)
        idx = top.indices.to(torch.int32).contiguous()
        wts = torch.softmax(top.values, dim=-1).float().contiguous()   # renormalised gate weights
        toks.append((x, idx, wts))
    # K4 at every instance (one launch with the step fence folded in, or begin_step + K4 on the
    # odd instances), then the expert stage, then K5
    for s in range(W):
        inst[s].dispatch(*toks[s], fused=(s % 2 == 0))
    rows = [inst[s].receive() for s in range(W)]
    per = E // W
    for s in range(W):
        sl = slice(s * per, (s + 1) * per)
        inst[s].expert_stage(rows[s][0], w_gate[sl], w_up[sl], w_down[sl])
    for s in range(W):
        inst[s].combine_put()
    for s in range(W):
        inst[s].combine_reduce()
    torch.cuda.synchronize()
    # received counts are what the gating implies
    for d in range(W):
        expect = [int(((toks[s][1] // per) == d).any(dim=1).sum().item()) for s in range(W)]
        assert rows[d][1].tolist() == expect
    port = oracle_lib.port()
    P = oracle_lib.P
    worst = 0.0
    for s in range(W):
        x, idx, wts = toks[s]
        M = x.shape[0]
        if M == 0:
            continue
        ref = np.zeros((M, H))
        assert port.dcpora_moe_layer_f64(M, H, I, E, k, P(_bits(x)), P(idx.cpu().numpy()), P(wts.cpu().numpy()),
                                         P(_bits(w_gate)), P(_bits(w_up)), P(_bits(w_down)), P(ref), 8) == 0
        got = inst[s].out[:M].cpu().double().numpy()
        rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
        worst = max(worst, rel.max())
    assert worst <= 2e-2, worst


@pytest.mark.parametrize("H,I", [(2048, 768), (7168, 2048)])
def test_real_expert_widths_at_cfg_token_counts(H, I):
    """cfg4 (Qwen3-30B-A3B: hidden 2,048, moe_intermediate 768) and cfg5 (DeepSeek-V3: hidden
    7,168, moe_intermediate 2,048) expert widths at the benched token count (128 per instance,
    8 instances, top-8), on a 16-expert subset (2 per rank) so the weights fit; the fp64 oracle
    checks 8 tokens of every instance (tokens are independent, so a subset is a full check of
    those tokens' dispatch -> experts -> combine)."""
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.moe import MoeInstance
    W, E, k, M, SUB = 8, 16, 8, 128, 8
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(H)
    inst = [MoeInstance(ctx, W, s, H, k, E, M) for s in range(W)]
    for s in range(W):
        for t in range(W):
            inst[s].set_peer_local(t, inst[t])
        inst[s].commit()
    w_gate = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_up = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_down = (torch.randn(E, H, I, generator=g, device=dev) / I ** 0.5).to(torch.bfloat16)
    toks = []
    for s in range(W):
        x = torch.randn(M, H, generator=g, device=dev).to(torch.bfloat16)
        top = torch.topk(torch.randn(M, E, generator=g, device=dev), k, dim=-1)
        toks.append((x, top.indices.to(torch.int32).contiguous(), torch.softmax(top.values, -1).float().contiguous()))
    for s in range(W):
        inst[s].dispatch(*toks[s])
    rows = [inst[s].receive() for s in range(W)]
    per = E // W
    for s in range(W):
        sl = slice(s * per, (s + 1) * per)
        inst[s].expert_stage(rows[s][0], w_gate[sl], w_up[sl], w_down[sl])
    for s in range(W):
        inst[s].combine_put()
    for s in range(W):
        inst[s].combine_reduce()
    torch.cuda.synchronize()
    for s in range(W):
        inst[s].status()
    port = oracle_lib.port()
    P = oracle_lib.P
    bg, bu, bd = _bits(w_gate), _bits(w_up), _bits(w_down)
    worst = 0.0
    for s in range(W):
        x, idx, wts = (t[:SUB] for t in toks[s])
        ref = np.zeros((SUB, H))
        assert port.dcpora_moe_layer_f64(SUB, H, I, E, k, P(_bits(x)), P(idx.cpu().numpy()), P(wts.cpu().numpy()),
                                         P(bg), P(bu), P(bd), P(ref), 16) == 0
        got = inst[s].out[:SUB].cpu().double().numpy()
        worst = max(worst, (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
    print(f"hidden {H} intermediate {I}: {W} x {M} tokens top-{k}, worst rel-L2 {worst:.2e}")
    assert worst <= 2e-2, worst
