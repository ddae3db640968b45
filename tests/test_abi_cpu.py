"""CPU-side checks of the C-ABI boundary: the library builds/loads and exports every
symbol include/powerfoam.h declares (no compute calls without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "powerfoam.h")).read()
    return sorted(set(re.findall(r"PF_API\s+[\w\s\*]+?\b(pf_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for core in ("pf_create_scene", "pf_render_forward", "pf_render_backward", "pf_destroy"):
        assert core in names
    assert len(names) >= 10


def test_library_exports_every_declared_symbol():
    import paper_2604_24994_b200 as pf
    L = pf.load_library()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(pf.EXPORTS)


def test_product_path_does_not_use_the_oracle():
    """The package never imports oracle/ and has no CPU fallback."""
    pkg = os.path.join(ROOT, "paper_2604_24994_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "liboracle" not in txt and "pf_oracle" not in txt, f


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2604_24994_b200 as pf
    t = torch.zeros(3)
    with pytest.raises(Exception):
        pf.Renderer(t.view(1, 3), t[:1], t[:1], t[:1], t.view(1, 3),
                    torch.zeros(2, dtype=torch.int64), torch.zeros(0, dtype=torch.int32))
