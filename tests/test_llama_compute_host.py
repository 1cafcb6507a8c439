"""Host logic of the Llama compute hook (paper_2411_00284_b200/llama_compute.py)
on CPU: per-parameter segments, the per-bucket forward / backward driver and
the re-gather swap of saved parameters (gathered parameters are
released after forward and re-gathered for backward), against plain torch
autograd of the same model.  No library calls: the slots are CPU tensors the
test fills the way the all-gather would.

The library's compute hook itself (fsdp_compute_hook) is exercised on the GPU
in tests/test_gpu_llama_compute.py."""
import types

import pytest
import torch

pytest.importorskip("paper_2411_00284_b200._lib", reason="libfsdp_b200.so not built")

from paper_2411_00284_b200 import _lib as L  # noqa: E402
from paper_2411_00284_b200 import llama_compute as LC  # noqa: E402
from paper_2411_00284_b200.harness import _carve  # noqa: E402
from workloads.shapes import ParamSpec  # noqa: E402


def mini_llama(layers=3, dim=256, heads=2, kv_heads=1, ffn=384, vocab=509):
    hd = LC.HEAD_DIM
    ps = [ParamSpec("tok_embeddings.weight", vocab, dim, 0)]
    for i in range(layers):
        pre, m = "layers.%d." % i, i + 1
        ps += [ParamSpec(pre + "attention_norm.weight", dim, 1, m),
               ParamSpec(pre + "attention.wq.weight", heads * hd, dim, m),
               ParamSpec(pre + "attention.wk.weight", kv_heads * hd, dim, m),
               ParamSpec(pre + "attention.wv.weight", kv_heads * hd, dim, m),
               ParamSpec(pre + "attention.wo.weight", dim, heads * hd, m),
               ParamSpec(pre + "ffn_norm.weight", dim, 1, m),
               ParamSpec(pre + "feed_forward.w1.weight", ffn, dim, m),
               ParamSpec(pre + "feed_forward.w3.weight", ffn, dim, m),
               ParamSpec(pre + "feed_forward.w2.weight", dim, ffn, m)]
    ps += [ParamSpec("norm.weight", dim, 1, layers + 1), ParamSpec("output.weight", vocab, dim, layers + 2)]
    return ps


def fake_rank(specs, fplan, bplan):
    """The attributes LlamaCompute reads from a RankState, world 1, on CPU."""
    full_numel = [s.dim0 * s.row_numel for s in specs]
    slot = max(_carve([full_numel[j] * 2 for j in b])[1] for b in list(fplan) + list(bplan))
    st = types.SimpleNamespace(
        specs=specs, world=1, rank=0, param_dtype=L.BF16, full_numel=full_numel,
        shard_offs=[0] * len(specs), shard_buf=torch.zeros(16, dtype=torch.uint8),
        full_slots=[torch.zeros(slot, dtype=torch.uint8) for _ in range(2)],
        grad_slots=[torch.zeros(slot, dtype=torch.uint8) for _ in range(2)],
        fwd=[types.SimpleNamespace(members=sorted(b)) for b in fplan],
        bwd=[types.SimpleNamespace(members=sorted(b)) for b in bplan])
    return st


class _NoStream:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@pytest.mark.parametrize("plan", ["per_block", "per_param", "mixed"])
def test_hooked_step_matches_autograd(plan, monkeypatch):
    torch.manual_seed(0)
    specs = mini_llama()     # 3 blocks: 6 per-block buckets, so a block's forward and backward slots differ
    P = len(specs)
    if plan == "per_block":
        mods = sorted({s.module_id for s in specs})
        fplan = [[j for j, s in enumerate(specs) if s.module_id == m] for m in mods]
    elif plan == "per_param":
        fplan = [[j] for j in range(P)]
    else:   # greedy-like: runs that cut across block boundaries
        cuts = [0, 1, 4, 7, 12, 13, 17, P - 2, P]
        fplan = [list(range(a, b)) for a, b in zip(cuts, cuts[1:])]
    bplan = [list(b) for b in reversed(fplan)]
    if plan == "mixed":     # backward buckets differ from the forward ones
        cuts = [0, 2, 9, 11, 15, P - 1, P]
        bplan = [list(range(a, b)) for a, b in zip(cuts, cuts[1:])][::-1]
    st = fake_rank(specs, fplan, bplan)
    params = []
    for s in specs:
        if LC.kind_of(s.name) in ("norm", "final_norm"):
            params.append(1.0 + 0.1 * torch.randn(s.dim0))
        else:
            params.append(0.05 * torch.randn(s.dim0, s.row_numel))
    params = [p.to(torch.bfloat16) for p in params]
    lc = LC.LlamaCompute(st, tokens=64, seed=3, norm_ones=False)
    monkeypatch.setattr(lc, "_stream", lambda handle: None)      # CPU: no streams
    monkeypatch.setattr(torch.cuda, "stream", lambda s: _NoStream())

    def gather(phase, b):
        for j, v in lc.views[phase][b].items():
            v.copy_(params[j].view(v.shape))

    def scribble(slot):
        st.full_slots[slot].fill_(0x7F)   # bf16 0x7F7F: large finite garbage

    for b in range(len(st.fwd)):
        gather(0, b)
        lc.hook(0, b, 0)
    loss = lc.state[0].clone()
    scribble(0)
    scribble(1)        # forward parameters released
    got = {}
    for b in range(len(st.bwd)):
        if b >= 2:
            scribble(b % 2)
        gather(1, b)   # re-gather into the backward slot
        lc.hook(1, b, 0)
        for j in st.bwd[b].members:   # grads of bucket b are final after its COMPUTE_B
            got[j] = lc.gviews[b][j].clone()
    assert not lc.saved
    ref_loss, ref = LC.reference_grads(specs, params, lc.ops.tokens, lc.ops.targets)
    assert torch.equal(loss, ref_loss)
    for j in range(P):
        g, r = got[j].float().reshape(-1), ref[j].float().reshape(-1)
        assert torch.isfinite(g).all()
        err = (g - r).norm() / max(r.norm(), 1e-30)
        assert err < 2e-2, (specs[j].name, float(err))


def test_kind_of_rejects_unknown_parameters():
    with pytest.raises(ValueError):
        LC.kind_of("fc0.weight")
