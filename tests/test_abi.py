"""C-ABI checks that need no GPU: libtide.so loads, exports every entry point
include/tide.h declares, and its host-only functions / argument validation
behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tide.h")


def _lib():
    from paper_2605_20179_b200 import _build
    _build.build()
    from paper_2605_20179_b200 import tide
    return tide


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tide_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("tide_moe_step", "tide_ctx_create", "tide_ctx_destroy", "tide_pack_expert",
              "tide_expert_bytes", "tide_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    tide = _lib()
    L = tide.lib()
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert set(tide.EXPORTED) <= set(declared_functions())


def test_library_is_sm100a_only():
    tide = _lib()
    assert tide.lib().tide_abi_version() == tide.ABI_VERSION
    assert tide.lib().tide_build_sm() == 100
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tide.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_expert_bytes():
    tide = _lib()
    d = tide.make_desc(256, 8, 2048, 512, 32)
    assert tide.expert_elems(d) == 3 * 2048 * 512
    assert tide.expert_bytes(d) == 3 * 2048 * 512 * 2
    d = tide.make_desc(16, 2, 64, 128, 8, tide.TIDE_F32)
    assert tide.expert_bytes(d) == 3 * 64 * 128 * 4


def test_argument_validation_without_device():
    """Bad descriptors are rejected before touching CUDA; a valid one fails
    cleanly (TIDE_ECUDA / TIDE_EUNSUPPORTED) when no sm_100 device exists."""
    tide = _lib()
    L = tide.lib()
    h = ctypes.c_void_p()
    bad = [tide.make_desc(0, 1, 64, 64, 8), tide.make_desc(8, 9, 64, 64, 8),
           tide.make_desc(8, 2, 100, 64, 8), tide.make_desc(8, 2, 64, 64, 0),
           tide.make_desc(8, 2, 64, 64, 2000)]
    for d in bad:
        rc = L.tide_ctx_create(ctypes.byref(d), 1, 4, 0, ctypes.byref(h))
        assert rc in (tide.TIDE_EINVAL, tide.TIDE_EUNSUPPORTED)
        assert L.tide_last_error()
    d = tide.make_desc(8, 2, 64, 64, 8)
    assert L.tide_ctx_create(ctypes.byref(d), 9, 4, 0, ctypes.byref(h)) == tide.TIDE_ECAPACITY
    assert L.tide_ctx_create(ctypes.byref(d), 0, 4, 0, ctypes.byref(h)) == tide.TIDE_ECAPACITY
    import torch
    if not torch.cuda.is_available():
        rc = L.tide_ctx_create(ctypes.byref(d), 2, 4, 0, ctypes.byref(h))
        assert rc == tide.TIDE_ECUDA and b"device" in L.tide_last_error()
    assert L.tide_moe_step(None, None, 0, None, None, None, 0, 1, 1, None, None, None, None,
                           None, None) == tide.TIDE_EINVAL
    # peer-memory EP: arguments checked before any CUDA call
    assert L.tide_ep_handle_bytes() == 64  # cudaIpcMemHandle_t
    d16 = tide.make_desc(16, 2, 64, 64, 8)
    assert L.tide_ctx_create_ep_p2p(ctypes.byref(d16), 0, 0, 16, ctypes.byref(h)) == \
        tide.TIDE_EUNSUPPORTED  # world > 8
    assert L.tide_ctx_create_ep_p2p(ctypes.byref(d16), 0, 0, 3, ctypes.byref(h)) == \
        tide.TIDE_EUNSUPPORTED  # 16 experts not divisible by 3
    assert L.tide_ctx_create_ep_p2p(ctypes.byref(d16), 0, 2, 2, ctypes.byref(h)) == tide.TIDE_EINVAL
    assert L.tide_ctx_ep_connect(None, None, None) == tide.TIDE_EINVAL
    assert L.tide_ctx_ep_export(None, None, None) == tide.TIDE_EINVAL
    v = ctypes.c_int32()
    assert L.tide_ctx_ep_error(None, ctypes.byref(v)) == tide.TIDE_EINVAL


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    """No CPU fallback: a missing libtide.so raises ImportError."""
    from paper_2605_20179_b200 import tide
    monkeypatch.setattr(tide, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(tide, "_lib", None)
    with pytest.raises(ImportError):
        tide.lib()


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's ctypes mirrors have the C structs' sizes (gcc on include/tide.h)."""
    import ctypes
    import subprocess
    tide = _lib()
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "tide.h"\nint main(void){printf("%zu %zu %zu %zu %zu\\n",'
                   'sizeof(tide_layer_desc), sizeof(tide_expert_weights), sizeof(tide_step_stats),'
                   'sizeof(tide_step_debug), sizeof(tide_phase_times)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(c) for c in (tide.LayerDesc, tide.ExpertWeights, tide.StepStats,
                                       tide.StepDebug, tide.PhaseTimes)]
    assert got == want
