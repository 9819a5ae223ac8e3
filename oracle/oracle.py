"""TEST INFRASTRUCTURE — ctypes wrapper of the CPU oracle (oracle/gt_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  It exposes the same handle interface as the product's
DeviceDag (`run`, `num_files`, `num_rules`, `grammar.dictionary`, `info`,
`dag_array`) so the reference-mirroring facade (paper_2106_06889_b200.tasks)
can render its results for comparison.

Parity pin: tests/test_oracle_golden.py (golden vectors from the reference).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2106_06889_b200._abi import (GtInfo, GtView, compact_from_view,
                                        raise_for_status)
from paper_2106_06889_b200.gtdc import GrammarView

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libgt_oracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.gto_open.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
        L.gto_open.restype = C.c_int
        L.gto_close.argtypes = [C.c_void_p]
        L.gto_info.argtypes = [C.c_void_p, C.POINTER(GtInfo)]
        L.gto_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.POINTER(C.c_void_p)]
        L.gto_run.restype = C.c_int
        L.gto_view.argtypes = [C.c_void_p, C.POINTER(GtView)]
        L.gto_free.argtypes = [C.c_void_p]
        L.gto_last_error.restype = C.c_char_p
        L.gto_dag_array.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]
        L.gto_dag_array.restype = C.c_int64
        _lib = L
    return _lib


class OracleDag:
    """CPU restatement of reference `build_dag` + engine (see gt_oracle.c)."""

    def __init__(self, blob: bytes, workers: int | None = None):
        self.workers = workers or os.cpu_count() or 1
        self._blob = bytes(blob)
        h = C.c_void_p()
        L = lib()
        st = L.gto_open(self._blob, len(self._blob), self.workers, C.byref(h))
        raise_for_status(st, L.gto_last_error().decode())
        self._h = h
        self.grammar = GrammarView(self._blob)
        inf = GtInfo()
        L.gto_info(self._h, C.byref(inf))
        self.info = inf.as_dict()

    @property
    def num_files(self) -> int:
        return self.info["num_files"]

    @property
    def num_rules(self) -> int:
        return self.info["num_rules"]

    def run(self, task: int, seq_len: int, strategy: int, file_set_width: int):
        L = lib()
        r = C.c_void_p()
        st = L.gto_run(self._h, task, seq_len, strategy, file_set_width, self.workers, C.byref(r))
        raise_for_status(st, L.gto_last_error().decode())
        try:
            v = GtView()
            L.gto_view(r, C.byref(v))
            return compact_from_view(v)
        finally:
            L.gto_free(r)

    def dag_array(self, name: str) -> np.ndarray:
        L = lib()
        n = L.gto_dag_array(self._h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.zeros(max(n, 1), dtype=np.int64)
        L.gto_dag_array(self._h, name.encode(), out.ctypes.data, len(out))
        return out[:n]

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().gto_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
