"""GPU parity against the reference's golden vectors (tests/golden).

Every fixture is loaded through the C-ABI (gt_open on cuda:0) and every
pinned output (six tasks, several sequence lengths, both strategies and
auto) must render byte-identically (sha256) to the reference's output; the
device-built DAG arrays must equal the reference build_dag arrays and the
level schedule must equal the reference's round schedule.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import expected, fixture_names, gtdc, output_jobs

pytestmark = pytest.mark.gpu

DAG_FIELDS = ["own_ids", "own_freqs", "own_off", "own_token_count", "sub_ids", "sub_freqs",
              "sub_off", "par_ids", "par_freqs", "par_off", "num_in_edge", "num_out_edge",
              "root_freq", "exp_len", "segment_token_counts"]


def arr_sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype="<i8")).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gt():
    import paper_2106_06889_b200 as gt
    return gt


@pytest.mark.parametrize("name", fixture_names())
def test_device_dag_matches_reference(gt, name):
    rec = expected()[name]["dag"]
    with gt.DeviceDag(gtdc(name)) as dag:
        info = dag.info
        assert info["num_rules"] == rec["num_rules"]
        assert info["num_files"] == rec["num_files"]
        assert info["depth"] == rec["depth"]
        assert info["total_elements"] == rec["total_elements"]
        assert info["words"] == rec["W"]
        assert info["td_levels"] == rec["td_rounds"]
        assert info["bu_levels"] == rec["bu_rounds"]
        for f in DAG_FIELDS:
            assert arr_sha(dag.dag_array(f)) == rec[f], f
        assert arr_sha(dag.dag_array("segments")) == rec["segments_sha"]
        assert arr_sha(dag.dag_array("td_level")) == rec["td_round"]
        assert arr_sha(dag.dag_array("bu_level")) == rec["bu_round"]


@pytest.mark.parametrize("name", fixture_names())
@pytest.mark.parametrize("strategy", ["auto", "topdown", "bottomup"])
def test_device_outputs_match_reference(gt, name, strategy):
    with gt.DeviceDag(gtdc(name)) as dag:
        for task, l, ent in output_jobs(name):
            out = gt.run_task(dag, task, gt.TraversalConfig(strategy=strategy), l)
            text = gt.render(out, dag.grammar.dictionary)
            got = hashlib.sha256(text.encode()).hexdigest()
            if got != ent["sha256"] and "text" in ent:
                pytest.fail(f"{task}@{l}: {gt.first_divergence(ent['text'], text)}")
            assert got == ent["sha256"], (task, l)


@pytest.mark.parametrize("name", fixture_names(kind="error"))
def test_device_errors_match_reference(gt, name):
    rec = expected()[name]
    exc = getattr(gt, rec["error"])
    with pytest.raises(exc) as info:
        gt.DeviceDag(gtdc(name))
    assert str(info.value) == rec["message"]
    assert info.value.exit_code == rec["exit_code"]


def test_unknown_task_and_bad_seq_len(gt):
    with gt.DeviceDag(gtdc("g1")) as dag:
        with pytest.raises(gt.UsageError, match="unknown task"):
            gt.run_task(dag, "frequencies", gt.TraversalConfig())
        with pytest.raises(gt.UsageError):
            gt.run_task(dag, "seqcount", gt.TraversalConfig(), 0)


def test_general_csr_path_matches_reference():
    """gt_open builds the own/sub CSR on the root-only fast path when no
    other body is longer than 32 symbols and redoes it on the general path
    otherwise; GT_CSR_GENERAL=1 forces the general path for every grammar
    (read once per process: a subprocess) — every Dag array still equal."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, GT_CSR_GENERAL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-x", "-q", "-p", "no:cacheprovider",
                        "-k", "test_device_dag_matches_reference"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
