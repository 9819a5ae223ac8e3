"""The task entry points take the reference's own `Dag` / `Grammar` objects
(SURVEY §8b): results equal those of the DeviceDag built from the same GTDC
bytes (a reference-shaped object is built here from the fixture; the real
reference's objects serialize to the same bytes, tests/test_reference_objects_cpu.py)."""

from __future__ import annotations

from types import SimpleNamespace

import pytest

from conftest import gtdc
from test_reference_objects_cpu import _fake_grammar
from test_shard_cpu import TASKS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["g1", "many_files_70", "composed_1"])
def test_reference_dag_object_runs_every_task(name):
    import paper_2106_06889_b200 as gt
    blob = gtdc(name)
    ref_dag = SimpleNamespace(grammar=_fake_grammar(blob))
    with gt.DeviceDag(blob) as dag:
        for task in TASKS:
            assert gt.run_task(ref_dag, task, gt.TraversalConfig()) == gt.run_task(dag, task, gt.TraversalConfig())
        assert gt.output_digest(ref_dag, "wordcount") == gt.output_digest(dag, "wordcount")
    d2 = gt.build_dag(ref_dag.grammar)
    try:
        assert d2.info["num_rules"] == len(ref_dag.grammar.bodies)
    finally:
        d2.close()
