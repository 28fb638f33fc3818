"""Config 1 stand-in: a Linear(16, 16) block with a debug print of the hidden
state and one tensor-dependent branch. GraphMend defers the print and
predicates the branch (2 sites found, 2 fixed)."""

import torch


class ToyBlock(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.fc = torch.nn.Linear(16, 16)

    def forward(self, x):
        h = self.fc(x)
        print("hidden:", h)
        if h.sum() > 0:
            y = h * 2
        else:
            y = h - 1
        return torch.relu(y)


torch.manual_seed(0)
model = ToyBlock()
compiled = torch.compile(model)
