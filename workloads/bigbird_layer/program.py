"""Config 2 as a full encoder layer: one BigBird-RoBERTa-base-shaped layer
(hidden 768, 12 heads of 64, block 64, intermediate 3072, post-LayerNorm,
GELU, seq 1024, batch 8).  The attention pattern is chosen from the score
statistics (block-sparse window + global block, or full), as in
workloads/bigbird_attn; both arms are softmaxes, so GraphMend predicates the
`if`, and the logger call is deferred.  The projections and the two batched
contractions run on cuBLAS; the softmax arms, the LayerNorms, the GELU and
the residual adds are the fused kernels' work."""

import logging

import torch

logger = logging.getLogger("bigbird_layer")


class BigBirdLayer(torch.nn.Module):
    def __init__(self, hidden=768, heads=12, block=64, seq=1024, intermediate=3072):
        super().__init__()
        self.query = torch.nn.Linear(hidden, hidden)
        self.key = torch.nn.Linear(hidden, hidden)
        self.value = torch.nn.Linear(hidden, hidden)
        self.output = torch.nn.Linear(hidden, hidden)
        self.attn_norm = torch.nn.LayerNorm(hidden, eps=1e-12)
        self.intermediate = torch.nn.Linear(hidden, intermediate)
        self.ffn_out = torch.nn.Linear(intermediate, hidden)
        self.out_norm = torch.nn.LayerNorm(hidden, eps=1e-12)
        self.heads = heads
        self.head_dim = hidden // heads
        blk = torch.arange(seq) // block
        window = (blk[:, None] - blk[None, :]).abs() <= 1
        glob = (blk[:, None] == 0) | (blk[None, :] == 0)
        self.register_buffer("mask_bias", torch.where(window | glob, 0.0, -10000.0))

    def forward(self, hidden):
        b, n, h = hidden.shape
        q = self.query(hidden).view(b, n, self.heads, self.head_dim).transpose(1, 2)
        k = self.key(hidden).view(b, n, self.heads, self.head_dim).transpose(1, 2)
        v = self.value(hidden).view(b, n, self.heads, self.head_dim).transpose(1, 2)
        scores = torch.matmul(q, k.transpose(-1, -2)) / 8.0
        bias = self.mask_bias
        logger.info("attention pattern selected")
        if scores.abs().mean() > 0.35:
            probs = torch.softmax(scores + bias, dim=-1)
        else:
            probs = torch.softmax(scores, dim=-1)
        ctx = torch.matmul(probs, v).transpose(1, 2).reshape(b, n, h)
        attn = self.attn_norm(self.output(ctx) + hidden)
        inter = torch.nn.functional.gelu(self.intermediate(attn))
        out = self.out_norm(self.ffn_out(inter) + attn)
        return out


torch.manual_seed(0)
model = BigBirdLayer()
compiled = torch.compile(model)
