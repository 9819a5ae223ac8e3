"""Native render + SHA-256 (render.cpp) against the reference-mirroring Python
`render` and hashlib, on the oracle's results for the golden fixtures (CPU:
the renderer is host code)."""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, expected, fixture_names, gtdc, output_jobs


def test_sha256_matches_hashlib():
    from paper_2106_06889_b200.native import sha256
    rng = np.random.default_rng(1)
    for n in (0, 1, 55, 56, 63, 64, 65, 119, 120, 127, 128, 1000, 4096 + 17, 1 << 20):
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert sha256(data) == hashlib.sha256(data).hexdigest(), n


def test_sha256_scalar_path_matches_hashlib():
    code = ("import hashlib,sys;sys.path.insert(0,%r);"
            "from paper_2106_06889_b200.native import sha256;"
            "d=bytes(range(256))*4099;"
            "assert sha256(d)==hashlib.sha256(d).hexdigest();print('ok')") % str(ROOT)
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "GT_SHA_SCALAR": "1"},
                         capture_output=True, text=True)
    assert out.stdout.strip() == "ok", out.stderr


@pytest.mark.parametrize("name", fixture_names(max_rules=20000))
def test_native_render_and_digest_match_reference(name):
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    from paper_2106_06889_b200.native import NativeDict
    blob = gtdc(name)
    ref = OracleDag(blob, workers=2)
    nd = NativeDict(blob)
    for task, l, ent in output_jobs(name):
        c = gt.run_compact(ref, task, gt.TraversalConfig(), l)
        text = gt.render(gt._abi.to_container(c), ref.grammar.dictionary)
        assert hashlib.sha256(text.encode()).hexdigest() == ent["sha256"]  # pinned
        assert nd.render(c) == text, (task, l)
        assert nd.digest(c) == (ent["sha256"], len(text.encode())), (task, l)
    ref.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g1", "many_files_70", "fuzz_05", "spill_70k_l4", "composed_3"])
def test_device_output_digest_is_reference_digest(name):
    import paper_2106_06889_b200 as gt
    with gt.DeviceDag(gtdc(name)) as dag:
        for task, l, ent in output_jobs(name):
            assert gt.output_digest(dag, task, gt.TraversalConfig(), l)[0] == ent["sha256"], (task, l)
            if "text" in ent:
                assert gt.render_native(dag, task, gt.TraversalConfig(), l) == ent["text"]
