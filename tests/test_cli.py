"""CLI contract (mirrors pkg/tests/test_cli.py): TSV on stdout, one JSON
manifest line on stderr with the sha256 outputDigest, exit codes of
errors.py.  Error-path tests run on CPU (the format check precedes any
device work); the analyze/verify/bench runs need the GPU."""

from __future__ import annotations

import json

import pytest

from conftest import expected, gtdc


def run_cli(capsys, *argv):
    from paper_2106_06889_b200.cli import main
    code = main([str(a) for a in argv])
    out, err = capsys.readouterr()
    return code, out, err


def test_missing_file_exit_2(tmp_path, capsys):
    code, _, err = run_cli(capsys, "analyze", tmp_path / "nope.gtdc", "wordcount")
    assert code == 2 and "gtadoc:" in err


def test_bad_magic_exit_3(tmp_path, capsys):
    p = tmp_path / "bad.gtdc"
    p.write_bytes(b"NOPE" + bytes(32))
    code, _, err = run_cli(capsys, "analyze", p, "wordcount")
    assert code == 3 and "bad magic" in err


def test_unknown_task_is_argparse_error():
    from paper_2106_06889_b200.cli import main
    with pytest.raises(SystemExit) as e:
        main(["analyze", "x.gtdc", "nosuchtask"])
    assert e.value.code == 2


def test_workers_env_must_be_integer(tmp_path, capsys, monkeypatch):
    p = tmp_path / "g1.gtdc"
    p.write_bytes(gtdc("g1"))
    monkeypatch.setenv("GTADOC_WORKERS", "three")
    code, _, err = run_cli(capsys, "analyze", p, "wordcount")
    assert code == 1 and "GTADOC_WORKERS" in err


@pytest.mark.gpu
@pytest.mark.parametrize("task", ["wordcount", "sort", "invertedindex", "termvector", "seqcount",
                                  "rankedinvertedindex"])
def test_analyze_tsv_and_manifest(task, tmp_path, capsys):
    p = tmp_path / "g1.gtdc"
    p.write_bytes(gtdc("g1"))
    code, out, err = run_cli(capsys, "analyze", p, task)
    assert code == 0
    ent = expected()["g1"]["outputs"][task if task not in ("seqcount", "rankedinvertedindex") else task + "@3"]
    manifest = json.loads(err.strip().splitlines()[-1])
    assert manifest["command"] == "analyze" and manifest["task"] == task and manifest["l"] == 3
    assert manifest["outputDigest"] == ent["sha256"]
    if "text" in ent:
        assert out == ent["text"]
    assert set(manifest["timings"]) >= {"initialization", "traversal"}


@pytest.mark.gpu
def test_analyze_out_file_and_verify_and_bench(tmp_path, capsys):
    p = tmp_path / "c.gtdc"
    p.write_bytes(gtdc("many_files_70"))
    code, out, err = run_cli(capsys, "analyze", p, "termvector", "--out", tmp_path / "tv.tsv")
    assert code == 0 and out == ""
    assert json.loads(err.strip().splitlines()[-1])["outputDigest"] == \
        expected()["many_files_70"]["outputs"]["termvector"]["sha256"]
    for task in ("wordcount", "invertedindex", "seqcount"):
        code, out, _ = run_cli(capsys, "verify", p, task)
        assert code == 0 and out.startswith(f"{task}\tok\t")
    code, out, _ = run_cli(capsys, "bench", p, "wordcount", "--repeat", "2", "--workers", "2")
    assert code == 0
    rows = dict(line.split("\t") for line in out.splitlines() if not line.startswith("#"))
    assert {"parallel-compressed", "sequential-compressed", "decompress-naive", "speedup-vs-sequential",
            "speedup-vs-naive"} <= set(rows)


@pytest.mark.gpu
def test_verify_and_bench_on_an_input_directory(tmp_path, capsys):
    """The reference's form (cli.py:137-193): a directory of text files,
    compressed first; verify counts the files' own tokens on the device."""
    import numpy as np
    rng = np.random.default_rng(7)
    d = tmp_path / "corpus"
    d.mkdir()
    vocab = [f"w{i}" for i in range(300)] + ["\u00e9t\u00e9", "na\u00efve"]
    for f in range(6):
        ids = np.minimum(rng.zipf(1.2, size=900 + 150 * f) - 1, len(vocab) - 1)
        (d / f"doc{f}.txt").write_text(" ".join(vocab[i] for i in ids) + ("\n" if f % 2 else ""))
    (d / "empty.txt").write_text("")
    for task in ("wordcount", "sort", "invertedindex", "termvector", "seqcount", "rankedinvertedindex"):
        for l in ((2, 4) if task in ("seqcount", "rankedinvertedindex") else (3,)):
            code, out, _ = run_cli(capsys, "verify", d, task, "--l", l)
            assert code == 0 and out.startswith(f"{task}\tok\t"), (task, l)
    code, out, _ = run_cli(capsys, "bench", d, "invertedindex", "--repeat", "1")
    assert code == 0 and "decompress-naive" in out


@pytest.mark.gpu
def test_count_tokens_matches_the_compressed_path():
    """gt_count_tokens on the files' token streams == every task's compressed
    result on the grammar of the same files."""
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200._abi import TASK_IDS
    from paper_2106_06889_b200.compress import compress_files, tokenize_files
    from test_shard_cpu import same_compact
    files = [("a.txt", b"a b a b c d a b"), ("b.txt", b"a b c"), ("c.txt", b""), ("d.txt", b"d d d c a b a b")]
    blob, _ = compress_files(files)
    toks, off = tokenize_files(files)
    assert off.tolist() == [0, 8, 11, 11, 19]
    with gt.DeviceDag(blob) as dag:
        for task in ("wordcount", "sort", "invertedindex", "termvector", "seqcount", "rankedinvertedindex"):
            for l in (1, 2, 3):
                same_compact(dag.count_tokens(TASK_IDS[task], l, toks, off), gt.run_compact(dag, task, gt.TraversalConfig(), l))


def test_compress_command_matches_reference_bytes(tmp_path, capsys):
    d = tmp_path / "g1"
    d.mkdir()
    (d / "A.txt").write_text("a b a b c")
    (d / "B.txt").write_text("a b c")
    out = tmp_path / "g1.gtdc"
    code, stdout, _ = run_cli(capsys, "compress", d, out)
    assert code == 0
    assert out.read_bytes() == gtdc("g1")
    rows = dict(line.split("\t") for line in stdout.splitlines())
    assert rows["files"] == "2" and rows["rules"] == "3" and rows["vocabulary"] == "3"


def test_compress_empty_dir_usage_error(tmp_path, capsys):
    empty = tmp_path / "empty"
    empty.mkdir()
    code, _, err = run_cli(capsys, "compress", empty, tmp_path / "x.gtdc")
    assert code == 1 and "no regular files" in err


def test_tokenize_gives_the_compressor_word_ids():
    """gt_tokenize's ids are the dictionary order of the GTDC gt_compress
    writes (first appearance), one stream per file, no splitters."""
    from paper_2106_06889_b200.compress import compress_files, tokenize_files
    from paper_2106_06889_b200.gtdc import read_dictionary
    files = [("A.txt", b"a b a b c"), ("B.txt", b"  a b\n c  x ")]
    toks, off = tokenize_files(files)
    words = read_dictionary(compress_files(files)[0]).words
    assert [words[i] for i in toks.tolist()] == ["a", "b", "a", "b", "c", "a", "b", "c", "x"]
    assert off.tolist() == [0, 5, 9]


def test_compress_invalid_utf8_ingest_error(tmp_path, capsys):
    corpus = tmp_path / "bad"
    corpus.mkdir()
    (corpus / "a.txt").write_bytes(b"ok bytes")
    (corpus / "b.txt").write_bytes(b"bad \xff\xfe here")
    code, _, err = run_cli(capsys, "compress", corpus, tmp_path / "x.gtdc")
    assert code == 2 and "b.txt" in err and "byte offset 4" in err
