"""C-ABI library: loads on a CPU-only box and exports every symbol include/lobe.h declares."""
import os
import re

from paper_2510_01767_b200 import lobe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lobe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lobe_[a-z_]+)\s*\(", src)) - {"lobe_objective_fn"})


def test_header_matches_binding_list():
    assert _declared() == sorted(lobe.EXPORTS)


def test_library_exports_every_symbol():
    L = lobe.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert "sm_100a" in lobe.version()


def test_no_device_fails_loudly_or_loads():
    """Without a GPU a compute call must fail with a CUDA status, never fall back."""
    import numpy as np
    import torch
    from synth import make_scene
    if torch.cuda.is_available():
        return
    s = make_scene("tiny")
    try:
        lobe.Scene(s, s)
    except lobe.LobeError as e:
        assert e.status == "CUDA"
    else:  # pragma: no cover
        raise AssertionError("compute succeeded without a CUDA device")
