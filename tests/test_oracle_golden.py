"""Pin the CPU oracle (oracle/gt_oracle.c) to the reference's golden vectors.

tests/golden/expected.json was produced by tools/make_golden.py running the
reference package itself; here the C restatement must reproduce every
rendered output byte-for-byte (sha256), every build_dag array, the
reference's round schedules, and every error class/message.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import expected, fixture_names, gtdc, output_jobs
from oracle.oracle import OracleDag
from paper_2106_06889_b200 import errors
from paper_2106_06889_b200.tasks import TraversalConfig, render, run_task

DAG_FIELDS = ["own_ids", "own_freqs", "own_off", "own_token_count", "sub_ids", "sub_freqs",
              "sub_off", "par_ids", "par_freqs", "par_off", "num_in_edge", "num_out_edge",
              "root_freq", "exp_len", "segment_token_counts"]


def arr_sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype="<i8")).tobytes()).hexdigest()


@pytest.mark.parametrize("name", fixture_names())
def test_oracle_dag_matches_reference(name):
    rec = expected()[name]["dag"]
    dag = OracleDag(gtdc(name), workers=2)
    info = dag.info
    assert info["num_rules"] == rec["num_rules"]
    assert info["num_files"] == rec["num_files"]
    assert info["depth"] == rec["depth"]
    assert info["total_elements"] == rec["total_elements"]
    assert info["words"] == rec["W"]
    for f in DAG_FIELDS:
        assert arr_sha(dag.dag_array(f)) == rec[f], f
    seg = dag.dag_array("segments")
    assert arr_sha(seg) == rec["segments_sha"]
    assert arr_sha(dag.dag_array("td_level")) == rec["td_round"]
    assert arr_sha(dag.dag_array("bu_level")) == rec["bu_round"]
    assert info["td_levels"] == rec["td_rounds"]
    assert info["bu_levels"] == rec["bu_rounds"]


@pytest.mark.parametrize("name", fixture_names())
@pytest.mark.parametrize("strategy", ["topdown", "bottomup", "auto"])
def test_oracle_outputs_match_reference(name, strategy):
    dag = OracleDag(gtdc(name), workers=4)
    for task, l, ent in output_jobs(name):
        out = run_task(dag, task, TraversalConfig(strategy=strategy), l)
        text = render(out, dag.grammar.dictionary)
        got = hashlib.sha256(text.encode()).hexdigest()
        if got != ent["sha256"] and "text" in ent:
            from paper_2106_06889_b200.tasks import first_divergence
            pytest.fail(f"{task}@{l}: {first_divergence(ent['text'], text)}")
        assert got == ent["sha256"], (task, l)
        assert text.count("\n") == ent["lines"]


@pytest.mark.parametrize("name", fixture_names(kind="error"))
def test_oracle_errors_match_reference(name):
    rec = expected()[name]
    exc = getattr(errors, rec["error"])
    with pytest.raises(exc) as info:
        OracleDag(gtdc(name), workers=1)
    assert str(info.value) == rec["message"]
    assert info.value.exit_code == rec["exit_code"]
