"""The C-ABI library builds, loads without a GPU, and exports every entry
point declared in include/slimfit_b200.h (no compute calls here)."""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "slimfit_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(sf_\w+)\s*\(", text, re.M)))


def test_header_declares_the_hot_path():
    names = declared_symbols()
    for must in ["sf_quant8", "sf_dequant8", "sf_prescale_exp", "sf_quant4_pack",
                 "sf_unpack4_dequant", "sf_prune_topk", "sf_restore", "sf_layer_distance",
                 "sf_layernorm_fwd", "sf_layernorm_bwd", "sf_softmax_fwd_q8", "sf_gelu_bwd_packed4"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2305_18513_b200 import _native as N
    if not os.path.exists(N.LIB_PATH):
        from paper_2305_18513_b200 import build
        build.build()
    exported = set(N.exported_symbols())
    declared = set(declared_symbols())
    assert declared <= set(N.SIGNATURES), declared - set(N.SIGNATURES)
    assert declared <= exported, declared - exported


def test_library_loads_and_reports_version():
    from paper_2305_18513_b200 import _native as N
    lib = N.load()
    assert lib.sf_abi_version() == 1
    assert lib.sf_strerror(1) == b"invalid argument"
    # argument validation happens before any device work: no GPU needed
    assert lib.sf_quant8(None, None, -1, 4, 1, None) == N.SF_EINVAL
    assert lib.sf_prune_topk(None, 0, 1, 1, None, None, None, None) == N.SF_EINVAL


def test_prescale_workspace_is_small():
    from paper_2305_18513_b200 import _native as N
    lib = N.load()
    assert 0 < lib.sf_prescale_workspace_bytes(50_331_648) < 1 << 16
    # staging slots for 5/32 of the elements as (value, index) pairs, 64 spare
    # slots per warp, the threshold-bin gather buffer: about 1.5 bytes per element
    assert lib.sf_prune_workspace_bytes(12_582_912) < 1.5 * 12_582_912 + (1 << 20)


def test_gemm_entry_validates_before_device_work():
    from paper_2305_18513_b200 import _native as N
    lib = N.load()
    # bad mode / negative sizes are rejected before cuBLASLt is touched
    assert lib.sf_gemm_f32(0, 0, 4, 4, 4, None, 4, 0, None, 4, 0, None, 4, 0, 1, None, 0.0, 7, None, 0,
                           None) == N.SF_EINVAL
    assert lib.sf_gemm_f32(0, 0, -1, 4, 4, None, 4, 0, None, 4, 0, None, 4, 0, 1, None, 0.0, 0, None, 0,
                           None) == N.SF_EINVAL
    # empty output: nothing to do
    assert lib.sf_gemm_f32(0, 0, 0, 4, 4, None, 4, 0, None, 4, 0, None, 4, 0, 1, None, 0.0, 0, None, 0,
                           None) == N.SF_OK


def test_gemm_operand_descriptors():
    """Transposed views fold into the cuBLAS op with the right leading
    dimension; collapsible batch dims give one stride (no copies)."""
    import torch
    from paper_2305_18513_b200 import gemm
    x = torch.zeros(6, 4)
    t, ld, batch, bs, tr = gemm._operand(x)
    assert (ld, batch, tr) == (4, 1, False) and t is x
    t, ld, batch, bs, tr = gemm._operand(x.t())
    assert (ld, batch, tr) == (4, 1, True) and t.data_ptr() == x.data_ptr()
    k = torch.zeros(2, 3, 5, 8)
    t, ld, batch, bs, tr = gemm._operand(k.transpose(-1, -2))
    assert (ld, batch, bs, tr) == (8, 6, 40, True) and t.data_ptr() == k.data_ptr()
    # a strided column slice keeps its leading dimension
    w = torch.zeros(10, 16)
    t, ld, batch, bs, tr = gemm._operand(w[:, :5])
    assert (ld, tr) == (16, False)
    # non-collapsible batch (permuted) is made contiguous
    p = torch.zeros(3, 2, 4, 5).permute(1, 0, 2, 3)
    t, ld, batch, bs, tr = gemm._operand(p)
    assert (batch, bs, tr) == (6, 20, False) and t.is_contiguous()
    for bad in ("fp64", "", "bf16"):
        with pytest.raises(ValueError):
            gemm.set_mode(bad)
