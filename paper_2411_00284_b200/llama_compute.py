"""Real Llama-3 compute plugged into the scheduled step.

The paper measures FSDP with the real model running between the collectives
(Tables 5/6); the bench's default compute is the calibrated proxy
K7.  ``LlamaCompute`` instead runs the Llama-3 layers themselves -- embedding,
RMSNorm, Q/K/V projections with RoPE and causal GQA attention (torch SDPA,
a library kernel), output projection, SwiGLU FFN, final norm, output layer and
cross-entropy loss -- on the parameters the library gathered, through the
schedule's compute hook (``fsdp_compute_hook``, include/fsdp.h): COMPUTE_F of a
bucket runs the forward of its members' ops, COMPUTE_B their backward, whose
weight gradients land in the bucket's full-gradient slots that PACK_RS then
averages.  Plumbing / measurement device only: PyTorch ops (cuBLAS GEMMs,
SDPA), none of the FSDP path.

Granularity is the parameter (reading O7 of SURVEY §8(c)): the op consuming
parameter j plus the parameterless ops that follow it (SDPA after wv, SiLU x
mul after w3, the loss after output) form segment j, so any plan (per-param,
per-block, greedy) maps onto the model.  Each segment runs under autograd with
its inputs detached; backward calls ``torch.autograd.grad`` per segment in
reverse order.  FSDP semantics: the forward's gathered parameters are
released (their slot is reused two buckets later) and the backward re-gathers
them into the backward bucket's slot, so every parameter tensor autograd saves
in forward is packed as a reference (saved_tensors_hooks) and unpacked as the
same view of the RE-GATHERED copy.
"""
import torch
import torch.nn.functional as Fn

from . import _lib as L
from .harness import _carve

HEAD_DIM = 128
ROPE_THETA = 500000.0   # Llama 3
NORM_EPS = 1e-5

_KINDS = (("tok_embeddings.weight", "emb"), ("attention_norm.weight", "norm"), ("attention.wq.weight", "wq"),
          ("attention.wk.weight", "wk"), ("attention.wv.weight", "wv"), ("attention.wo.weight", "wo"),
          ("ffn_norm.weight", "norm"), ("feed_forward.w1.weight", "w1"), ("feed_forward.w3.weight", "w3"),
          ("feed_forward.w2.weight", "w2"), ("norm.weight", "final_norm"), ("output.weight", "out"))


def kind_of(name):
    for suffix, k in _KINDS:
        if name == suffix or name.endswith("." + suffix):
            return k
    raise ValueError("LlamaCompute: no Llama op consumes parameter %r" % name)


def rope_tables(T, device):
    inv = 1.0 / (ROPE_THETA ** (torch.arange(0, HEAD_DIM, 2, device=device, dtype=torch.float32) / HEAD_DIM))
    ang = torch.outer(torch.arange(T, device=device, dtype=torch.float32), inv)
    return torch.cos(ang), torch.sin(ang)      # [T, HEAD_DIM / 2]


def apply_rope(x, cos, sin):
    """x [T, H, HEAD_DIM] bf16: rotate (even, odd) pairs by position angle (fp32 math)."""
    xf = x.float().unflatten(-1, (-1, 2))
    a, b = xf[..., 0], xf[..., 1]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.stack((a * c - b * s, a * s + b * c), dim=-1).flatten(-2).to(x.dtype)


class LlamaOps:
    """The per-parameter segments of a Llama-3 model: forward(kind, state, W)
    -> state.  State between segments: (x,) on the residual stream; (x, h)
    after a norm; (x, h, q), (x, h, q, k) inside attention; (x, a) after
    attention; (x, h, g) inside the FFN, (x, m) after SiLU(g) * (h W3^T);
    (h,) after the final norm; (loss,) after the output layer."""

    def __init__(self, tokens, targets):
        self.tokens, self.targets = tokens, targets
        self.cos, self.sin = rope_tables(tokens.numel(), tokens.device)

    def attention(self, q, k, v):
        T = q.shape[0]
        H, KV = q.shape[1] // HEAD_DIM, k.shape[1] // HEAD_DIM
        q = apply_rope(q.view(T, H, HEAD_DIM), self.cos, self.sin)
        k = apply_rope(k.view(T, KV, HEAD_DIM), self.cos, self.sin)
        v = v.view(T, KV, HEAD_DIM)
        rep = H // KV            # grouped-query attention: each KV head serves `rep` query heads
        k = k.repeat_interleave(rep, dim=1)
        v = v.repeat_interleave(rep, dim=1)
        o = Fn.scaled_dot_product_attention(q.transpose(0, 1)[None], k.transpose(0, 1)[None],
                                            v.transpose(0, 1)[None], is_causal=True)
        return o[0].transpose(0, 1).reshape(T, H * HEAD_DIM)

    def forward(self, kind, st, W):
        if kind == "emb":
            return (Fn.embedding(self.tokens, W),)
        if kind == "norm":
            x, = st
            return x, Fn.rms_norm(x, (x.shape[-1],), W.reshape(-1), NORM_EPS)
        if kind == "final_norm":
            x, = st
            return (Fn.rms_norm(x, (x.shape[-1],), W.reshape(-1), NORM_EPS),)
        if kind == "wq":
            x, h = st
            return x, h, Fn.linear(h, W)
        if kind == "wk":
            x, h, q = st
            return x, h, q, Fn.linear(h, W)
        if kind == "wv":
            x, h, q, k = st
            return x, self.attention(q, k, Fn.linear(h, W))
        if kind in ("wo", "w2"):
            x, a = st
            return (x + Fn.linear(a, W),)
        if kind == "w1":
            x, h = st
            return x, h, Fn.linear(h, W)
        if kind == "w3":
            x, h, g = st
            return x, Fn.silu(g) * Fn.linear(h, W)
        if kind == "out":
            h, = st
            return (Fn.cross_entropy(Fn.linear(h, W).float(), self.targets),)
        raise ValueError(kind)


def flops_per_step(specs, T):
    """Model FLOPs of one forward + backward (2 T |W| forward per linear, 2x
    that backward; causal attention 2 T^2 d_head H forward (QK^T + PV, half
    masked), 2.5x that backward)."""
    f = 0
    for s in specs:
        k = kind_of(s.name)
        if k in ("wq", "wk", "wv", "wo", "w1", "w3", "w2", "out"):
            f += 6 * T * s.dim0 * s.row_numel
        if k == "wv":
            H = next(p.dim0 for p in specs if p.name == s.name.replace("wv", "wq")) // HEAD_DIM
            f += 3.5 * 2 * T * T * HEAD_DIM * H
    return f


class LlamaCompute:
    """Compute hook of one rank's scheduled step (RankState ``st``) at T
    tokens: ``st.step(..., hook=lc.hook)``.  Tokens and targets are seeded
    random ids (synthetic data)."""

    def __init__(self, st, tokens, seed=11, norm_ones=True):
        if st.param_dtype != L.BF16:
            raise ValueError("LlamaCompute needs bf16 parameters")
        self.st, self.T = st, int(tokens)
        self.kinds = [kind_of(s.name) for s in st.specs]
        dev = st.shard_buf.device
        g = torch.Generator(device=dev).manual_seed(seed)
        vocab = next(s.dim0 for s, k in zip(st.specs, self.kinds) if k == "emb")
        self.ops = LlamaOps(torch.randint(0, vocab, (self.T,), generator=g, device=dev),
                            torch.randint(0, vocab, (self.T,), generator=g, device=dev))
        if norm_ones:   # Llama init: norm weights 1.0 (the rank's valid rows of each norm shard)
            c = [-(-s.dim0 // st.world) for s in st.specs]
            for j, (s, k) in enumerate(zip(st.specs, self.kinds)):
                if k in ("norm", "final_norm"):
                    v = max(0, min(s.dim0 - st.rank * c[j], c[j]))
                    o = st.shard_offs[j]
                    st.shard_buf[o:o + 2 * v].view(torch.bfloat16).fill_(1.0)
        # views of every member's gathered parameter / full gradient, per phase and bucket
        slot_of = getattr(st, "full_slot_index", lambda phase, b: b % 2)
        self.views = (self._views(st.fwd, st.full_slots, lambda b: slot_of(0, b)),
                      self._views(st.bwd, st.full_slots, lambda b: slot_of(1, b)))
        ng = getattr(st, "n_grad_slots", 2)
        self.gviews = self._views(st.bwd, st.grad_slots, lambda b: b % ng)
        self.saved = {}
        self.gstate = None
        self.state = ()
        self.cur_w = None
        self._streams = {}
        self.flops = flops_per_step(st.specs, self.T)
        if dev.type == "cuda":
            # the fills above ran on torch's current stream; the step's streams are not ordered after it
            torch.cuda.synchronize(dev)

    def _views(self, buckets, slots, slot_of):
        out = []
        for b, bk in enumerate(buckets):
            offs, _ = _carve([self.st.full_numel[j] * 2 for j in bk.members])
            d = {}
            for j, o in zip(bk.members, offs):
                s = self.st.specs[j]
                v = slots[slot_of(b)][o:o + 2 * s.dim0 * s.row_numel].view(torch.bfloat16)
                d[j] = v.view(s.dim0, s.row_numel) if s.row_numel > 1 else v
            out.append(d)
        return out

    def _stream(self, handle):
        s = self._streams.get(handle)
        if s is None:
            s = self._streams[handle] = torch.cuda.ExternalStream(handle)
        return s

    # ------------------------------------------------------------- hook
    def hook(self, phase, bucket, stream):
        with torch.cuda.stream(self._stream(stream)):
            if phase == 0:
                self._forward(bucket)
            else:
                self._backward(bucket)

    def _forward(self, b):
        bk = self.st.fwd[b]
        if b == 0:
            self.state, self.saved, self.gstate = (), {}, None
        for j in bk.members:
            W = self.views[0][b][j].detach().requires_grad_(True)
            wptr, woff = W.untyped_storage().data_ptr(), W.storage_offset()

            def pack(t, j=j, wptr=wptr, woff=woff):
                if t.untyped_storage().data_ptr() == wptr and t.dtype == torch.bfloat16:
                    return ("W", j, t.size(), t.stride(), t.storage_offset() - woff)
                return t

            ins = tuple(t.detach().requires_grad_(True) for t in self.state)
            with torch.enable_grad(), torch.autograd.graph.saved_tensors_hooks(pack, self._unpack):
                outs = self.ops.forward(self.kinds[j], ins, W)
            self.saved[j] = (ins, W, outs)
            self.state = tuple(o.detach() for o in outs)

    def _unpack(self, x):
        if isinstance(x, tuple) and len(x) == 5 and x[0] == "W":
            _, j, size, stride, delta = x
            base = self.cur_w[j]        # the re-gathered parameter (backward slot)
            return torch.as_strided(base, size, stride, base.storage_offset() + delta)
        return x

    def _backward(self, b):
        bk = self.st.bwd[b]
        self.cur_w = self.views[1][b]
        for j in sorted(bk.members, reverse=True):
            ins, W, outs = self.saved.pop(j)
            if self.gstate is None:       # the loss: d loss / d loss = 1
                self.gstate = (torch.ones_like(outs[0]),)
            pairs = [(o, g) for o, g in zip(outs, self.gstate) if g is not None and o.requires_grad]
            need = list(ins) + [W]
            grads = torch.autograd.grad([o for o, _ in pairs], need, [g for _, g in pairs], allow_unused=True)
            dW = grads[-1]
            gv = self.gviews[b][j]
            if dW is None:
                gv.zero_()
            else:
                gv.copy_(dW.view(gv.shape))
            self.gstate = tuple(grads[:-1])
        self.cur_w = None


def reference_grads(specs, params, tokens, targets):
    """Plain torch autograd of the same model over full parameters (the check
    of the hooked step): params[j] bf16 tensors; returns (loss, [dW_j])."""
    ops = LlamaOps(tokens, targets)
    ws = [p.detach().clone().requires_grad_(True) for p in params]
    st = ()
    for j, s in enumerate(specs):
        st = ops.forward(kind_of(s.name), st, ws[j])
    loss, = st
    loss.backward()
    return loss.detach(), [w.grad for w in ws]


