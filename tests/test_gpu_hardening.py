"""predicate hardening.

The reference copies predicate source verbatim (transform.py:386-388) and
reports these sites fixed with residual 0, but at runtime
  * `p and q` on tensor predicates calls Tensor.__bool__ (a host sync), and
  * `not p` hands torch.where a Python bool and raises (torch 2.11).
The B200 lowering evaluates and/or/not of 0-d bool predicates on the device.
The checker is the ORIGINAL (untransformed) program on CPU, whose `if`
semantics the rewrite is meant to preserve."""

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import compile_program

ORIGINAL = '''import torch

def f(x):
    h = x * 2
    if (h.sum() > 0) and (h.max() < 5):
        y = h + 1
    else:
        y = h - 1
    if not (y.mean() > 0):
        z = y * 3
    else:
        z = y
    return z

fc = torch.compile(f)
'''

# what the reference fix_file returns for ORIGINAL (generated in the build
# container with /root/reference; 2 found, 2 fixed, predicted residual 0)
TRANSFORMED = '''import torch

def f(x):
    h = x * 2
    __gm_pred_0 = (h.sum() > 0) and (h.max() < 5)
    __gm_then_y_0 = h + 1
    __gm_else_y_0 = h - 1
    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
    __gm_pred_1 = not (y.mean() > 0)
    __gm_then_z_0 = y * 3
    __gm_else_z_0 = y
    z = torch.where(__gm_pred_1, __gm_then_z_0, __gm_else_z_0)
    return z

fc = torch.compile(f)
'''


def test_reference_rewrite_fails_at_runtime_on_cpu():
    """The defect being hardened: the transformed `not` predicate raises."""
    fn = orc.reference_callable(TRANSFORMED, "f")
    with pytest.raises(TypeError):
        fn(torch.full((64,), -1.0))


@pytest.mark.gpu
@pytest.mark.parametrize("fill", [1.0, 4.0, -1.0, None])
def test_hardened_predicates_match_original(fill):
    x = torch.randn(8, 1024, 768) if fill is None else torch.full((8, 1024, 768), fill)
    ref = orc.reference_callable(ORIGINAL, "f")(x.clone())
    ex, mod, low = compile_program(TRANSFORMED, "f")
    out = ex(x.cuda())
    torch.cuda.synchronize()
    info = ex.info()[0]
    assert info.mode == "graph" and info.host_syncs == 0, info
    assert low.regions[0].stats.launches >= 1
    torch.testing.assert_close(out.cpu(), ref, rtol=1e-5, atol=1e-5)
