"""SURVEY §8f rank 3 stand-in: a BigBird-RoBERTa-base-shaped layer (hidden
768, seq 1024, batch 8) whose data-dependent branch picks between two dense
projections — a "local" one for dense activations and a "global" one
otherwise — so BOTH arms of the predicated block hold a GEMM
(transform.py:272 admits torch-rooted calls such as torch.matmul in arms;
the rewrite evaluates both, transform.py:404-412). The query projection is a
Linear on cuBLAS; the arm projections read plain local names, as the purity
gate requires (attributes are refused inside arms)."""

import logging

import torch

logger = logging.getLogger("gemm_arms")


class GemmArmLayer(torch.nn.Module):
    def __init__(self, hidden=768):
        super().__init__()
        self.query = torch.nn.Linear(hidden, hidden)
        self.w_local = torch.nn.Parameter(torch.randn(hidden, hidden) * hidden ** -0.5)
        self.b_local = torch.nn.Parameter(torch.randn(hidden) * 0.02)
        self.w_global = torch.nn.Parameter(torch.randn(hidden, hidden) * hidden ** -0.5)
        self.b_global = torch.nn.Parameter(torch.randn(hidden) * 0.02)

    def forward(self, hidden):
        q = self.query(hidden)
        wl, bl, wg, bg = self.w_local, self.b_local, self.w_global, self.b_global
        logger.info("projection selected")
        if q.abs().mean() > 0.4:
            ctx = torch.matmul(q, wl) + bl
        else:
            ctx = torch.matmul(q, wg) * 0.5 + bg
        return ctx + hidden


torch.manual_seed(0)
model = GemmArmLayer()
compiled = torch.compile(model)
