"""Shared test fixtures.  GPU tests are marked `gpu` and only run on a B200."""

from __future__ import annotations

import gzip
import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@lru_cache(maxsize=None)
def expected() -> dict:
    return json.loads((GOLDEN / "expected.json").read_text())["fixtures"]


@lru_cache(maxsize=None)
def gtdc(name: str) -> bytes:
    return gzip.decompress((GOLDEN / "grammars" / f"{name}.gtdc.gz").read_bytes())


def fixture_names(kind=None, max_rules=None, exclude=()):
    out = []
    for name, rec in sorted(expected().items()):
        if name in exclude:
            continue
        if kind == "error":
            if rec["kind"] == "error":
                out.append(name)
            continue
        if rec["kind"] == "error":
            continue
        if max_rules is not None and rec["dag"]["num_rules"] > max_rules:
            continue
        out.append(name)
    return out


def output_jobs(name):
    """(task, seq_len, expected-entry) for every pinned output of a fixture."""
    rec = expected()[name]
    jobs = []
    for key, ent in sorted(rec["outputs"].items()):
        if "@" in key:
            task, l = key.split("@")
            jobs.append((task, int(l), ent))
        else:
            jobs.append((key, 3, ent))
    return jobs
