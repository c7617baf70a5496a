"""The C-ABI boundary without a GPU: libkvpr.so loads, exports every symbol
include/kvpr.h declares, the ctypes struct layout equals the C layout, the
SASS is Blackwell-native, and the product path has no CPU fallback."""

from __future__ import annotations

import ctypes
import re
import shutil
import subprocess

import pytest

from paper_2411_17089_b200 import _lib

from .conftest import ROOT

HEADER = ROOT / "include" / "kvpr.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \t*]*?\b(kvpr_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert names, "no declarations parsed from include/kvpr.h"
    for n in names:
        assert hasattr(lib, n), f"libkvpr.so does not export {n}"
    assert set(names) == set(_lib.EXPORTS), "ctypes binding and header disagree"


def test_version_and_error_string(lib):
    assert lib.kvpr_version() == 2
    assert isinstance(_lib.last_error(), str)


def test_ctypes_struct_layout_matches_c(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "kvpr.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(kvpr_epilogue),"
        " offsetof(kvpr_epilogue, seg_width), offsetof(kvpr_epilogue, ld), offsetof(kvpr_epilogue, seg),"
        " offsetof(kvpr_epilogue, scale), offsetof(kvpr_epilogue, scale_cols), offsetof(kvpr_epilogue, flags),"
        " sizeof(kvpr_out_seg)); return 0;}\n")
    src.write_text(src.read_text().replace(
        "return 0;}",
        'printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(kvpr_decoder_desc), offsetof(kvpr_decoder_desc, eps),'
        " offsetof(kvpr_decoder_desc, embed), offsetof(kvpr_decoder_desc, ws_bytes),"
        " offsetof(kvpr_decoder_desc, d2h_stream), sizeof(kvpr_layer_desc));"
        ' printf("%zu %zu\\n", offsetof(kvpr_decoder_desc, chunk_rows), offsetof(kvpr_decoder_desc, chunk_wave));'
        ' printf("%zu %zu\\n", offsetof(kvpr_decoder_desc, recompute_stream), offsetof(kvpr_decoder_desc, zero_copy));'
        ' printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(kvpr_layer_tail_desc), offsetof(kvpr_layer_tail_desc, scale),'
        ' offsetof(kvpr_layer_tail_desc, q), offsetof(kvpr_layer_tail_desc, lnx_ld),'
        ' offsetof(kvpr_layer_tail_desc, host_hi), offsetof(kvpr_layer_tail_desc, ws_bytes));'
        ' return 0;}'))
    exe = tmp_path / "layout"
    subprocess.run([gcc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    E, D = _lib.Epilogue, _lib.DecoderDesc
    want = [ctypes.sizeof(E), E.seg_width.offset, E.ld.offset, E.seg.offset, E.scale.offset, E.scale_cols.offset,
            E.flags.offset, ctypes.sizeof(_lib.OutSeg),
            ctypes.sizeof(D), D.eps.offset, D.embed.offset, D.ws_bytes.offset, D.d2h_stream.offset,
            ctypes.sizeof(_lib.LayerDesc), D.chunk_rows.offset, D.chunk_wave.offset,
            D.recompute_stream.offset, D.zero_copy.offset]
    T = _lib.LayerTailDesc
    want += [ctypes.sizeof(T), T.scale.offset, T.q.offset, T.lnx_ld.offset, T.host_hi.offset, T.ws_bytes.offset]
    assert got == want


def test_sass_is_tcgen05_tma(lib):
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    try:
        out = subprocess.run([cuobjdump, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True,
                             timeout=120).stdout
    except (FileNotFoundError, subprocess.TimeoutExpired):
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in out, "no tcgen05.mma in SASS"
    assert "UTMALDG" in out, "no TMA loads in SASS"
    assert "LDTM" in out, "no tcgen05.ld in SASS"
    # warp-level mma.sync only in the fused small-batch layer tail (6-21 weight rows per CTA: the dense
    # GEMMs -- K1, prefill projections and attention, decode projections -- are tcgen05) and its
    # bit-equality probe
    hmma_funcs = []
    for block in out.split("Function : ")[1:]:
        name = block.split("\n", 1)[0].strip()
        if "HMMA" in block.replace("UTCHMMA", ""):
            hmma_funcs.append(name)
    assert hmma_funcs and all("layer_tail" in n or "mma_linear_probe" in n for n in hmma_funcs), hmma_funcs


def test_missing_library_fails_loudly(tmp_path):
    saved = _lib._lib
    _lib._lib = None
    try:
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            _lib.load(tmp_path / "nope.so")
    finally:
        _lib._lib = saved


def test_product_path_rejects_cpu_tensors():
    import torch

    from paper_2411_17089_b200 import kernels

    x = torch.zeros(4, 2, 64, dtype=torch.float16)
    w = torch.zeros(128, 64, dtype=torch.float16)
    with pytest.raises(ValueError, match="CUDA"):
        kernels.recompute_kv(x, w, None, torch.zeros(4, 2, 2, 64, dtype=torch.float16), 2, 0, 2)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2411_17089_b200"
    for p in pkg.rglob("*.py"):
        text = p.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, flags=re.M), f"{p} imports the oracle"


def test_recompute_tile_choice(lib):
    """K1's tile (host-side, no GPU): the CTA pair when 256x256 tiles fill the 74 SM pairs, else the
    widest 1-CTA tile that still covers half the SMs; the bench labels its roofline line with it."""
    assert lib.kvpr_recompute_tile(32, 296, 4096, 148) == 512   # config 2 chunk: 37 x 32 pair tiles
    assert lib.kvpr_recompute_tile(4, 250, 768, 148) == 128     # config 1: 8 m-blocks x 12 = 96 tiles
    assert lib.kvpr_recompute_tile(1, 1, 256, 148) == 32
    assert lib.kvpr_recompute_tile(0, 10, 256, 148) == 0
