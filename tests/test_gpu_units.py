"""The reference's own unit fixtures (pkg/tests/fixtures/units/*.py, its
transform tests' equivalence cases, test_transform.py:281-379) through the
B200 path on branch-forcing inputs, against CPU eager of the same transformed
text: elif chains, nested ifs, if-without-else (prior value), augmented
assignments, intra-arm dependencies, multiple targets, multi-return deferral,
tensor prints (including torch's summarised repr), item reads, dynamic-shape
ops, loops and impure branches (the last ones stay eager: syncs or immediate
side effects)."""

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import compile_program, harness
from parity import assert_parity


def full(shape, v):
    return torch.full(shape if isinstance(shape, tuple) else (shape,), float(v))


BIG = (8, 1024, 768)
CASES = {
    # name: (callable, [arg tuples], expect_graph)
    "tensor_branch": ("f", [(full(6, 4.0), torch.randn(6)), (full(6, -1.0), torch.randn(6)),
                            (torch.randn(BIG) + 0.01, torch.randn(BIG))], True),
    "augassign_branch": ("bump", [(full(4, 1.5),), (full(4, -1.5),), (torch.randn(BIG),)], True),
    "intra_arm_dep": ("chainy", [(full(4, 3.0),), (full(4, -3.0),), (torch.randn(7, 13),)], True),
    "nested_if_branch": ("fold", [(full(4, 9.0),), (full(4, 1.0),), (full(4, -1.0),), (full(BIG, 0.5),)], True),
    "elif_chain": ("route", [(full(4, 30.0),), (full(4, 0.0),), (full(4, -30.0),), (torch.randn(BIG),)], True),
    "if_no_else": ("clip", [(full(4, 3.0),), (full(4, 0.25),), (torch.randn(BIG),)], True),
    "multi_target": ("pair", [(full(4, 2.0),), (full(4, -2.0),), (torch.randn(1001),)], True),
    "debug_print_mid": ("fn", [(torch.tensor([0.5, -1.0, 2.0]),), (torch.randn(2000),), (torch.randn(5, 300),)],
                        True),
    "multi_return_defer": ("split", [(torch.randn(5), True), (torch.randn(5), False)], True),
    "mixed_breaks": ("steps", [(full(4, 3.0),), (full(4, -3.0),)], True),
    "entry_module_compile": ("net", [(full(4, 1.0),), (full(4, -1.0),)], True),
    "shadowing": ("shade", [(full(4, 1.0),), (full(4, -1.0),)], True),
    "static_attr_guard": ("sized", [(torch.randn(12),), (torch.randn(5),)], True),
    "taint_kill": ("steady", [(torch.randn(4),)], True),
    "item_access": ("scale", [(torch.randn(64),)], True),
    "dynamic_shape_op": ("pick", [(torch.randn(64),), (torch.randn(BIG),)], True),
    "helper_call": ("outer", [(torch.randn(4),)], True),
    "loop_tensor_cond": ("drain", [(full(4, 2.0),)], False),
    "impure_branch": ("head", [(full(4, 5.0),), (full(4, -5.0),)], False),
    "print_in_branch": ("noisy", [(full(4, 1.0),), (full(4, -1.0),)], False),
    "unsupported_region": ("guarded", [(full(4, 1.0),), (full(4, -1.0),)], False),
}


@pytest.mark.gpu
@pytest.mark.parametrize("unit", sorted(CASES))
def test_unit_fixture_on_b200(programs, unit):
    fn_name, arg_sets, expect_graph = CASES[unit]
    prog = programs[f"unit:{unit}"]
    text = prog["transformed"]
    for args in arg_sets:
        ref_fn = orc.reference_callable(text, fn_name)
        ref, ref_text = orc.call_captured(ref_fn, list(args))
        ex, mod, low = compile_program(text, fn_name)
        dev_args = [a.cuda() if torch.is_tensor(a) else a for a in args]
        out, out_text = harness.call_captured(ex, dev_args)
        assert out_text == ref_text, (unit, out_text, ref_text)
        if isinstance(ref, torch.Tensor):
            assert_parity(out, ref, torch.float32, what=unit)
        else:
            assert out == ref
        info = ex.info()[0]
        if expect_graph:
            assert info.mode == "graph" and info.host_syncs == 0, (unit, info)
        else:
            assert info.mode == "eager", (unit, info)
