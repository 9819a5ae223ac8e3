"""bench.py host logic on CPU: SURVEY §8(d) algorithmic bytes, and the
reference arm (the oracle restatement) end to end at a small scale with the
same config dict as our arm."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

# the C2 bench corpus (BENCH_r01 config) and its inverted-index records
C2 = {"num_rules": 840001, "sub_pairs": 1118513, "own_pairs": 2044250, "root_len": 54663,
      "num_words": 100000, "num_files": 16, "total_elements": 3414928, "words": 166733450, "depth": 24}
O_II = 543223


def test_alg_bytes_follow_survey_8d():
    R, Es, Eo, L0, V, F = 840001, 1118513, 2044250, 54663, 100000, 16
    wc = 8 * Es + 8 * Eo + 4 * L0 + 8 * (R + 1) * 2 + 16 * R + 8 * V
    ii = 8 * Es + 8 * Eo + 4 * L0 + 16 * R + 4 * (F + 1) + O_II * (4 + 4)
    assert bench.alg_bytes_task("wordcount", C2, 0) == wc
    assert bench.alg_bytes_task("invertedindex", C2, O_II) == ii
    fused, per_task = bench.alg_bytes_step(C2, O_II)
    assert per_task == wc + ii
    assert abs(per_task / 1e6 - 96.5) < 0.1  # 53.2 MB + 43.3 MB
    # one shared pass reads the DAG once: fewer compulsory bytes than the sum
    assert fused == per_task - (8 * Es + 8 * Eo + 4 * L0)
    assert fused < per_task


def test_reference_arm_small(tmp_path):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--scale", "0.002",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "words/s"
    assert line["warmup"] == 1 and line["steps"] == 2
    cfg = line["config"]
    assert cfg["workload"].startswith("c2:") and cfg["parallelism"] == "1 shard" and cfg["l2"] == bench.L2_NOTE
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
