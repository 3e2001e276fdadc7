"""The C-ABI library builds, loads without a GPU and exports every function
include/tlk.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2410_22254_b200 import runtime as rt

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "tlk.h")


def declared():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tlk_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared()
    assert "tlk_open" in names and "tlk_run" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = rt.lib()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(rt.EXPORTS)


def test_pure_calls_work_without_gpu():
    lib = rt.lib()
    assert lib.tlk_abi_version() == 1
    info = rt.model_info(rt.MODEL_CNN)
    assert info.param_count == 1_199_882 and info.param_stride % 64 == 0
    assert info.flops_per_sample == 6 * (26 * 26 * 32 * 9 + 24 * 24 * 64 * 288 + 9216 * 128 + 1280)
    # layout table agrees with the oracle's restatement
    from oracle import models

    for model in (rt.MODEL_MLP, rt.MODEL_CNN):
        lay, count, stride = models.layout(model)
        assert [(off, t.count, t.fan_in) for t, off in lay] == rt.model_tensors(model)
        assert rt.model_info(model).param_stride == stride


def test_open_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        return
    ctx = ctypes.c_void_p()
    rc = rt.lib().tlk_open(0, ctypes.byref(ctx))
    assert rc != 0 and rt.lib().tlk_last_error()
