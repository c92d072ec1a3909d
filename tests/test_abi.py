"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and rejects bad scalar arguments before touching the device."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2303_14335_b200 as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "mpld.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpld_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = mp.lib()
    names = _header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(L, name), name
        assert isinstance(getattr(L, name), ctypes._CFuncPtr)
    assert sorted(mp.EXPORTS) == names


def test_version_and_kernel_names():
    assert mp.version() == "0.1.0"
    L = mp.lib()
    names = [L.mpld_kernel_name(i).decode() for i in range(L.mpld_kernel_count())]
    assert "mpld_exact_cover_search" in names and "mpld_simplify_components" in names


@pytest.mark.parametrize("k,alpha,msg", [(1, 0.1, "k must"), (5, 0.1, "k must"), (3, -0.5, "alpha"),
                                         (3, 0.0005, "multiple"), (3, 2000.0, "alpha")])
def test_scalar_argument_errors(k, alpha, msg):
    z = np.zeros(4, np.int32)
    with pytest.raises(mp.MPLDError) as ei:
        mp.mpld_decompose(3, z, np.zeros(0, np.int32), z, np.zeros(0, np.int32), k, alpha)
    assert ei.value.code == 1 and msg in str(ei.value)


def test_stats_layout_matches_header():
    src = open(os.path.join(ROOT, "include", "mpld.h")).read()
    enum = re.findall(r"MPLD_STAT_([A-Z_]+)\s*=\s*(\d+)", src)
    idx = {name: int(v) for name, v in enum}
    assert idx["LEN"] == len(mp.STAT_NAMES)
    order = ["COMPONENTS", "HIDDEN", "ROUNDS", "MAX_COMP", "STEPS", "TRUNCATED", "ERROR", "LAUNCHES", "MAX_STEPS",
             "SPILL_REFUSED"]
    assert [idx[o] for o in order] == list(range(len(order)))


def test_product_path_does_not_import_oracle():
    """The binding and the CUDA sources never reference oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2303_14335_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_host_binding_rejects_wrong_element_types():
    """Host entry points: torch tensors of another element type and output
    arrays of another element type are rejected before the C ABI is called."""
    import torch
    z = np.zeros(4, np.int32)
    with pytest.raises(TypeError):
        mp.mpld_decompose_batch(np.array([0, 3], np.int32), 3, torch.zeros(4, dtype=torch.int64),
                                np.zeros(0, np.int32), z, np.zeros(0, np.int32), 3, 0.1)
    with pytest.raises(TypeError):
        mp.mpld_decompose_batch(np.array([0, 3], np.int32), 3, z, np.zeros(0, np.int32), z, np.zeros(0, np.int32),
                                3, 0.1, out_colors=np.zeros(3, np.int64))
