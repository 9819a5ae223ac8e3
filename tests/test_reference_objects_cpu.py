"""The drop-in boundary accepts the reference's own objects (SURVEY §8b:
"dag may be a reference Dag or the new device-resident handle"): a reference
`Grammar` / `Dag` is serialized back to GTDC bytes exactly as the reference's
serialize_grammar writes them (grammar.py:164-174).  CPU-only checks; the
reference package is imported from /root/reference when present (this
container), never on the GPU box."""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import pytest

from conftest import gtdc

REF = "/root/reference/pkg/src"


def _fake_grammar(blob):
    """A reference-shaped Grammar (dictionary.words, num_splitters, bodies)
    parsed from GTDC bytes with the package's own header reader."""
    import struct

    import numpy as np
    nw, ns, R = struct.unpack_from("<III", blob, 5)
    pos, words = 17, []
    for _ in range(nw):
        (n,) = struct.unpack_from("<I", blob, pos)
        words.append(blob[pos + 4:pos + 4 + n].decode("utf-8"))
        pos += 4 + n
    bodies = []
    for _ in range(R):
        (n,) = struct.unpack_from("<I", blob, pos)
        bodies.append(np.frombuffer(blob, dtype="<u4", count=n, offset=pos + 4).astype(np.int64))
        pos += 4 + 4 * n
    return SimpleNamespace(dictionary=SimpleNamespace(words=words, num_splitters=ns), bodies=bodies)


@pytest.mark.parametrize("name", ["g1", "many_files_70", "composed_1", "spill_70k_l4"])
def test_reference_shaped_grammar_and_dag_serialize_to_the_same_bytes(name):
    from paper_2106_06889_b200.device import gtdc_of
    blob = gtdc(name)
    g = _fake_grammar(blob)
    assert gtdc_of(g) == blob
    assert gtdc_of(SimpleNamespace(grammar=g)) == blob  # a Dag carries its grammar
    assert gtdc_of(b"not a grammar") is None


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
@pytest.mark.parametrize("name", ["g1", "many_files_70", "composed_1"])
def test_real_reference_objects_serialize_to_the_fixture(name):
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    try:
        from gtadoc.dag import build_dag
        from gtadoc.grammar import deserialize_grammar
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference not importable: {e}")
    from paper_2106_06889_b200.device import gtdc_of
    blob = gtdc(name)
    g = deserialize_grammar(blob)
    assert gtdc_of(g) == blob
    assert gtdc_of(build_dag(g)) == blob
