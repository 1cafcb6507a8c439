"""Parameter shapes in forward-use order (reading G5).

Llama 3.1 dims from Table 2: layers / model dim / FFN dim / heads.
Vocabulary 128,256, 8 KV heads and head_dim 128 are NOT in the paper; they are
the Llama 3 family values (reading G23).  Output weight untied from the
embedding (G24).  A parameter of shape [d, ...] is described by its dim 0 ``d``
and the product of its other dims ``row_numel`` (1 for 1-D tensors).

module_id drives manual wrapping: embedding 0, transformer block
i -> i + 1, final norm L + 1, output L + 2.
"""
from collections import namedtuple

ParamSpec = namedtuple("ParamSpec", "name dim0 row_numel module_id")

LLAMA_CONFIGS = {
    # name: (layers, dim, ffn_dim, heads)   -- Table 2
    "8b": (32, 4096, 14336, 32),
    "70b": (80, 8192, 28672, 64),
    "405b": (126, 16384, 53248, 128),
}
VOCAB = 128256
N_KV_HEADS = 8
HEAD_DIM = 128


def llama(name="8b", n_layers=None, with_embeddings=True):
    layers, dim, ffn, heads = LLAMA_CONFIGS[name]
    if n_layers is not None:
        layers = n_layers
    kv = N_KV_HEADS * HEAD_DIM
    ps = []
    if with_embeddings:
        ps.append(ParamSpec("tok_embeddings.weight", VOCAB, dim, 0))
    for i in range(layers):
        m = i + 1
        pre = "layers.%d." % i
        ps += [
            ParamSpec(pre + "attention_norm.weight", dim, 1, m),
            ParamSpec(pre + "attention.wq.weight", heads * HEAD_DIM, dim, m),
            ParamSpec(pre + "attention.wk.weight", kv, dim, m),
            ParamSpec(pre + "attention.wv.weight", kv, dim, m),
            ParamSpec(pre + "attention.wo.weight", dim, heads * HEAD_DIM, m),
            ParamSpec(pre + "ffn_norm.weight", dim, 1, m),
            ParamSpec(pre + "feed_forward.w1.weight", ffn, dim, m),
            ParamSpec(pre + "feed_forward.w3.weight", ffn, dim, m),
            ParamSpec(pre + "feed_forward.w2.weight", dim, ffn, m),
        ]
    if with_embeddings:
        ps.append(ParamSpec("norm.weight", dim, 1, layers + 1))
        ps.append(ParamSpec("output.weight", VOCAB, dim, layers + 2))
    return ps


def toy_mlp():
    """BASELINE.json configs[0]: 4-layer MLP 33 -> 71 -> 57 -> 43 -> 13 with bias;
    8 tensors, 9,584 elements, every dim 0 odd (padding at N = 2)."""
    dims = [33, 71, 57, 43, 13]
    ps = []
    for i in range(4):
        ps.append(ParamSpec("fc%d.weight" % i, dims[i + 1], dims[i], i))
        ps.append(ParamSpec("fc%d.bias" % i, dims[i + 1], 1, i))
    return ps


def numel(ps):
    return sum(p.dim0 * p.row_numel for p in ps)


# Tensor-parallel plan for the 2-D DP x TP mesh, TorchTitan-style:
# column-parallel weights are split on dim 0 (output features), row-parallel
# ones on dim 1 (input features), the embedding on dim 0 (vocabulary), norms
# replicated.  Only shapes live here; slicing values is the oracle's job.
TP_AXIS = {"attention.wq.weight": 0, "attention.wk.weight": 0, "attention.wv.weight": 0,
           "feed_forward.w1.weight": 0, "feed_forward.w3.weight": 0, "output.weight": 0,
           "tok_embeddings.weight": 0, "attention.wo.weight": 1, "feed_forward.w2.weight": 1}


def tp_axis(spec):
    """0 / 1: the dim the TP plan splits; None: replicated over TP."""
    for suffix, ax in TP_AXIS.items():
        if spec.name.endswith(suffix):
            return ax
    return None


def tp_local(specs, tp):
    """The TP-local shapes of `specs` on a TP group of size `tp` (every split
    dim divisible by tp for the Llama shapes at tp <= 8)."""
    out = []
    for p in specs:
        ax = tp_axis(p)
        if ax == 0:
            assert p.dim0 % tp == 0
            out.append(p._replace(dim0=p.dim0 // tp))
        elif ax == 1:
            assert p.row_numel % tp == 0
            out.append(p._replace(row_numel=p.row_numel // tp))
        else:
            out.append(p)
    return out
