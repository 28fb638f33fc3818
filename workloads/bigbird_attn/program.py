"""Config 2 with its attention: one BigBird-RoBERTa-base-shaped
self-attention layer (hidden 768, 12 heads of 64, block 64, seq 1024,
batch 8), the scores materialised as [8, 12, 1024, 1024].  The attention
pattern is chosen from the score statistics: spread-out scores take the
block-sparse pattern (a sliding window of 3 blocks plus the global first
block, as an additive mask), otherwise full attention.  Both arms are a
softmax over the key dim, so GraphMend predicates the `if` (the arms are
pure torch calls, transform.py:265-289) and both softmaxes would run
eagerly; the logger call is deferred to the epilogue.  The projections and
the two batched contractions run on cuBLAS."""

import logging

import torch

logger = logging.getLogger("bigbird_attn")


class BigBirdAttnLayer(torch.nn.Module):
    def __init__(self, hidden=768, heads=12, block=64, seq=1024):
        super().__init__()
        self.query = torch.nn.Linear(hidden, hidden)
        self.key = torch.nn.Linear(hidden, hidden)
        self.value = torch.nn.Linear(hidden, hidden)
        self.output = torch.nn.Linear(hidden, hidden)
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
        out = self.output(ctx)
        return out + hidden


torch.manual_seed(0)
model = BigBirdAttnLayer()
compiled = torch.compile(model)
