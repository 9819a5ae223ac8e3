"""CPU-side checks of the C-ABI library and the host facade (no GPU needed)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "gtadoc_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(gt_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2106_06889_b200.build import build
    lib_path = build()
    lib = ctypes.CDLL(str(lib_path))
    syms = declared_symbols()
    assert "gt_open" in syms and "gt_run" in syms and len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    lib.gt_abi_version.restype = ctypes.c_int
    assert lib.gt_abi_version() == 3


def test_python_facade_lists_the_header_exports():
    from paper_2106_06889_b200.device import EXPORTS
    assert sorted(EXPORTS) == declared_symbols()


def test_library_links_only_cuda_runtime_and_system_libs():
    import subprocess
    from paper_2106_06889_b200.build import build
    out = subprocess.run(["ldd", str(build())], capture_output=True, text=True).stdout
    assert "oracle" not in out
    assert "torch" not in out


def test_traversal_config_validation():
    from paper_2106_06889_b200 import TraversalConfig, UsageError
    with pytest.raises(UsageError):
        TraversalConfig(workers=0)
    with pytest.raises(UsageError):
        TraversalConfig(chunk_factor=0)
    with pytest.raises(UsageError):
        TraversalConfig(strategy="sideways")


def test_render_and_first_divergence_match_reference_contract():
    from paper_2106_06889_b200.gtdc import Dictionary
    from paper_2106_06889_b200.tasks import (RankedInvertedIndex, SequenceCounts, TermVectors,
                                            WordCounts, first_divergence, render)
    d = Dictionary(words=["a", "b", "c"], num_splitters=2)
    assert render(WordCounts({1: 3, 0: 3, 2: 2}), d) == "a\t3\nb\t3\nc\t2\n"
    tv = TermVectors([[(0, 2), (1, 2), (2, 1)], [(0, 1), (1, 1), (2, 1)]])
    assert render(tv, d).splitlines()[0] == "0\ta\t2"
    sc = SequenceCounts([{(0, 1, 0): 1, (1, 0, 1): 1, (0, 1, 2): 1}, {(0, 1, 2): 1}])
    assert render(sc, d) == "0\ta b a\t1\n0\ta b c\t1\n0\tb a b\t1\n1\ta b c\t1\n"
    rii = RankedInvertedIndex({(0, 1, 2): [(0, 1), (1, 1)], (0, 1, 0): [(0, 1)]})
    assert render(rii, d) == "a b a\t0:1\na b c\t0:1\t1:1\n"
    assert first_divergence("a\t1\nb\t2\n", "a\t1\nb\t3\n") == "line 2: expected 'b\\t2', got 'b\\t3'"
    assert first_divergence("a\t1\n", "a\t1\n") is None


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2106_06889_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
    for p in (pkg / "csrc").glob("*"):
        assert "gt_oracle" not in p.read_text(), p


def test_view_layout_matches_the_header_and_narrow_ids_decode():
    """ABI 3: the ctypes GtView mirrors gt_view field for field (offsets from
    the header's declaration order), and a view whose ids travel 1 or 2 bytes
    wide decodes to the same ids as the u32 form."""
    import ctypes as C
    import re
    from pathlib import Path

    import numpy as np

    from paper_2106_06889_b200._abi import GtView, compact_from_view
    hdr = (Path(__file__).resolve().parents[1] / "include" / "gtadoc_b200.h").read_text()
    body = hdr[hdr.index("typedef struct gt_view {"):hdr.index("} gt_view;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)  # (comments)
    names = re.findall(r"\b(\w+);", body)
    assert [f[0] for f in GtView._fields_] == names
    ids = np.array([3, 0, 7, 255, 1], dtype=np.uint32)
    cnt = np.array([5, 4, 3, 2, 1], dtype=np.uint64)
    for width, dt in ((4, np.uint32), (2, np.uint16), (1, np.uint8)):
        v = GtView()
        v.task = 0  # wordcount
        v.n = len(ids)
        a = ids.astype(dt)
        if width == 4:
            v.id = a.ctypes.data_as(C.POINTER(C.c_uint32))
        else:
            v.id_narrow = a.ctypes.data
            v.id_bytes = width
        v.count = cnt.ctypes.data_as(C.POINTER(C.c_uint64))
        c = compact_from_view(v)
        assert c.id.tolist() == ids.tolist() and c.count.tolist() == cnt.tolist()
