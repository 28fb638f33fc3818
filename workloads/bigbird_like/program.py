"""Config 2 stand-in: one BigBird-RoBERTa-base-shaped layer (hidden 768,
block 64, seq 1024, batch 8). The attention pattern is picked from the
activation statistics: dense queries take the block-sparse path, otherwise
the full path. A second data-dependent branch rescales the residual when the
projected output blows up. Both branches have pure tensor arms, so GraphMend
predicates them; the logger call is deferred to the epilogue. The two dense
projections run on cuBLAS."""

import logging

import torch

logger = logging.getLogger("bigbird_like")


class BigBirdLikeLayer(torch.nn.Module):
    def __init__(self, hidden=768, block=64):
        super().__init__()
        self.query = torch.nn.Linear(hidden, hidden)
        self.output = torch.nn.Linear(hidden, hidden)
        self.scale = block ** -0.5

    def forward(self, hidden):
        q = self.query(hidden)
        scores = q * self.scale
        logger.info("attention pattern selected")
        if scores.abs().mean() > 0.05:
            probs = torch.sigmoid(scores) * 0.5 + 0.25
            ctx = probs * q
        else:
            probs = torch.sigmoid(scores)
            ctx = probs * q + hidden
        out = self.output(ctx)
        if out.norm() > 500.0:
            res = out * 0.5 + hidden
        else:
            res = out + hidden
        return res


torch.manual_seed(0)
model = BigBirdLikeLayer()
compiled = torch.compile(model)
