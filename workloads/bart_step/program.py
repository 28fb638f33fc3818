"""Config 4 stand-in: one BART-base-shaped decoder step for a batch of 32
sequences (d_model 768, ffn 3072, one new token per sequence). Per-stage
logging sits between the tensor stages; GraphMend hoists all three calls to
the epilogue so the step is one captured graph. The dense layers run on
cuBLAS."""

import logging

import torch

logger = logging.getLogger("bart_step")


class DecoderStep(torch.nn.Module):
    def __init__(self, d_model=768, ffn=3072):
        super().__init__()
        self.q_proj = torch.nn.Linear(d_model, d_model)
        self.fc1 = torch.nn.Linear(d_model, ffn)
        self.fc2 = torch.nn.Linear(ffn, d_model)

    def forward(self, hidden):
        logger.info("decoder step start")
        q = self.q_proj(hidden)
        h = torch.tanh(q) * 0.5 + hidden
        logger.debug("self-attention done")
        f = torch.relu(self.fc1(h))
        out = self.fc2(f) + h
        logger.info("decoder step done, %d layers", 1)
        return out * 0.5


torch.manual_seed(0)
model = DecoderStep()
compiled = torch.compile(model)
