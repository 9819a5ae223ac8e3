"""DeviceDag: the device-resident counterpart of the reference `Dag`.

`build_dag(blob)` mirrors `deserialize_grammar` + `build_dag`
(`src/grammar.py:193-228`, `src/dag.py:131-230`) through `gt_open`; the
handle exposes what `render` and the task facade need (`num_files`,
`num_rules`, `grammar.dictionary`) plus `info` (R, E, W, depth, ...).

The CUDA library is mandatory: if libgtadoc_b200.so is missing or no CUDA
device is present, `lib()` raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from ._abi import GtInfo, GtView, compact_from_view, raise_for_status
from .errors import UsageError, ResourceError
from .gtdc import GrammarView

LIB_PATH = Path(__file__).resolve().parent / "libgtadoc_b200.so"
EXPORTS = ("gt_abi_version", "gt_last_error", "gt_open", "gt_info_get", "gt_run",
           "gt_result_view", "gt_result_free", "gt_close", "gt_device_word_counts",
           "gt_dag_array", "gt_flush_l2", "gt_sync", "gt_profile", "gt_profile_report",
           "gt_set_files", "gt_assemble_counts", "gt_dict_open", "gt_dict_close", "gt_render_view",
           "gt_free_text", "gt_digest_view", "gt_sha256", "gt_table_add_batch", "gt_run_naive",
           "gt_compress", "gt_compress_free", "gt_compress_last_error", "gt_run_many", "gt_clone",
           "gt_device_count", "gt_sum_word_counts", "gt_count_tokens", "gt_tokenize")
_lib = None


def lib():
    """Load libgtadoc_b200.so (fails loudly when absent)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ResourceError(f"{LIB_PATH} is missing: run `python -m paper_2106_06889_b200.build`")
        L = C.CDLL(str(LIB_PATH))
        L.gt_abi_version.restype = C.c_int
        L.gt_last_error.restype = C.c_char_p
        L.gt_open.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_uint64, C.c_uint64,
                              C.POINTER(C.c_void_p)]
        L.gt_open.restype = C.c_int
        L.gt_info_get.argtypes = [C.c_void_p, C.POINTER(GtInfo)]
        L.gt_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.gt_run.restype = C.c_int
        L.gt_run_many.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_void_p)]
        L.gt_run_many.restype = C.c_int
        L.gt_result_view.argtypes = [C.c_void_p, C.POINTER(GtView)]
        L.gt_result_free.argtypes = [C.c_void_p]
        L.gt_close.argtypes = [C.c_void_p]
        L.gt_device_word_counts.argtypes = [C.c_void_p]
        L.gt_device_word_counts.restype = C.c_void_p
        L.gt_dag_array.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]
        L.gt_dag_array.restype = C.c_int64
        L.gt_flush_l2.argtypes = [C.c_void_p]
        L.gt_sync.argtypes = [C.c_void_p]
        L.gt_profile.argtypes = [C.c_void_p, C.c_int]
        L.gt_profile_report.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        L.gt_profile_report.restype = C.c_int64
        L.gt_set_files.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.gt_dict_open.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.gt_dict_close.argtypes = [C.c_void_p]
        L.gt_render_view.argtypes = [C.c_void_p, C.POINTER(GtView), C.POINTER(C.c_void_p),
                                     C.POINTER(C.c_uint64)]
        L.gt_free_text.argtypes = [C.c_void_p]
        L.gt_digest_view.argtypes = [C.c_void_p, C.POINTER(GtView), C.c_char_p, C.POINTER(C.c_uint64)]
        L.gt_sha256.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p]
        L.gt_compress.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_uint64), C.c_void_p]
        L.gt_compress_free.argtypes = [C.c_void_p]
        L.gt_compress_last_error.restype = C.c_char_p
        L.gt_run_naive.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.gt_table_add_batch.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                         C.c_void_p, C.c_void_p]
        L.gt_assemble_counts.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
        L.gt_clone.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.gt_clone.restype = C.c_int
        L.gt_device_count.restype = C.c_int
        L.gt_sum_word_counts.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int]
        L.gt_sum_word_counts.restype = C.c_int
        L.gt_count_tokens.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.POINTER(C.c_void_p)]
        L.gt_count_tokens.restype = C.c_int
        L.gt_tokenize.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p), C.c_void_p]
        L.gt_tokenize.restype = C.c_int
        _lib = L
    return _lib


def device_count() -> int:
    """Visible CUDA devices (gt_device_count)."""
    return int(lib().gt_device_count())


def _err() -> str:
    return lib().gt_last_error().decode(errors="replace")


class DeviceDag:
    """Grammar loaded, validated and flattened on one CUDA device."""

    def __init__(self, blob, device: int = 0, file_lo: int = 0,
                 file_hi: int = (1 << 64) - 1):
        """`blob`: GTDC bytes, or (host_pointer, nbytes) of a (pinned) buffer."""
        self._h = None
        if isinstance(blob, tuple):
            ptr, nbytes = blob
            src = C.cast(C.c_void_p(ptr), C.c_char_p)
            self._blob = None
        else:
            self._blob = bytes(blob)
            src, nbytes = self._blob, len(self._blob)
        h = C.c_void_p()
        L = lib()
        st = L.gt_open(src, nbytes, device, file_lo, file_hi, C.byref(h))
        raise_for_status(st, _err())
        self._h = h
        self.device = device
        self.grammar = GrammarView(self._blob) if self._blob is not None else None
        self._info = None

    @property
    def info(self) -> dict:
        """gt_info_get.  The first call completes the derived DAG arrays
        (exp_len, heights, W, segment token counts), which gt_open leaves to
        the first task that reads them."""
        if self._info is None:
            inf = GtInfo()
            raise_for_status(lib().gt_info_get(self._h, C.byref(inf)), _err())
            self._info = inf.as_dict()
        return self._info

    def refresh_info(self) -> dict:
        """Re-read gt_info (info is a snapshot: device_bytes and load_flags
        change when a run builds lazy structures, e.g. the contraction)."""
        self._info = None
        return self.info

    @property
    def num_files(self) -> int:
        return self.info["num_files"]

    @property
    def num_rules(self) -> int:
        return self.info["num_rules"]

    def run(self, task: int, seq_len: int, strategy: int, file_set_width: int):
        L = lib()
        r = C.c_void_p()
        st = L.gt_run(self._h, task, seq_len, strategy, file_set_width, C.byref(r))
        raise_for_status(st, _err())
        try:
            v = GtView()
            L.gt_result_view(r, C.byref(v))
            return compact_from_view(v)
        finally:
            L.gt_result_free(r)

    def run_many(self, tasks, seq_len: int, strategy: int, file_set_width: int):
        """gt_run_many: several tasks in one call (word count + inverted index
        share one device pass); returns one Compact per task."""
        rs = self.run_many_raw(tasks, seq_len, strategy, file_set_width)
        try:
            return [compact_from_view(v) for _, v in rs]
        finally:
            for r, _ in rs:
                self.free_raw(r)

    def run_many_raw(self, tasks, seq_len: int = 3, strategy: int = 0, file_set_width: int = 64):
        """gt_run_many returning [(result handle, view)] without copying."""
        L = lib()
        n = len(tasks)
        ids = (C.c_int * n)(*tasks)
        outs = (C.c_void_p * n)()
        st = L.gt_run_many(self._h, ids, n, seq_len, strategy, file_set_width, outs)
        raise_for_status(st, _err())
        res = []
        for i in range(n):
            v = GtView()
            L.gt_result_view(outs[i], C.byref(v))
            res.append((C.c_void_p(outs[i]), v))
        return res

    def run_raw(self, task: int, seq_len: int = 3, strategy: int = 0, file_set_width: int = 64):
        """gt_run returning (result handle, view) without copying the arrays;
        caller frees with `free_raw`.  Used by the e2e bench leg."""
        L = lib()
        r = C.c_void_p()
        st = L.gt_run(self._h, task, seq_len, strategy, file_set_width, C.byref(r))
        raise_for_status(st, _err())
        v = GtView()
        L.gt_result_view(r, C.byref(v))
        return r, v

    @staticmethod
    def free_raw(r) -> None:
        lib().gt_result_free(r)

    def run_naive(self, task: int, seq_len: int = 3):
        """gt_run_naive: decompress-then-count (verification ground truth)."""
        L = lib()
        r = C.c_void_p()
        raise_for_status(L.gt_run_naive(self._h, task, seq_len, C.byref(r)), _err())
        try:
            v = GtView()
            L.gt_result_view(r, C.byref(v))
            return compact_from_view(v)
        finally:
            L.gt_result_free(r)

    def count_tokens(self, task: int, seq_len: int, tokens: np.ndarray, file_off: np.ndarray):
        """gt_count_tokens: the task counted on the given per-file token
        streams (the plain text), by the device counting stage only."""
        L = lib()
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        file_off = np.ascontiguousarray(file_off, dtype=np.uint64)
        r = C.c_void_p()
        raise_for_status(L.gt_count_tokens(self._h, task, seq_len, tokens.ctypes.data, file_off.ctypes.data,
                                           len(file_off) - 1, C.byref(r)), _err())
        try:
            v = GtView()
            L.gt_result_view(r, C.byref(v))
            return compact_from_view(v)
        finally:
            L.gt_result_free(r)

    def set_files(self, file_lo: int, file_hi: int) -> None:
        """Restrict subsequent runs to files [file_lo, file_hi) (gt_set_files)."""
        raise_for_status(lib().gt_set_files(self._h, file_lo, file_hi), _err())

    def assemble_counts(self, dev_ptr: int, task: int):
        """wordcount/sort result from a dense u64[V] device vector (gt_assemble_counts)."""
        L = lib()
        r = C.c_void_p()
        raise_for_status(L.gt_assemble_counts(self._h, task, C.c_void_p(dev_ptr), C.byref(r)), _err())
        try:
            v = GtView()
            L.gt_result_view(r, C.byref(v))
            return compact_from_view(v)
        finally:
            L.gt_result_free(r)

    def device_word_counts_ptr(self) -> int:
        return lib().gt_device_word_counts(self._h) or 0

    def clone(self, device: int) -> "DeviceDag":
        """gt_clone: this DAG replicated onto `device` by peer copies (built
        once, broadcast over NVLink); same file range, same grammar view."""
        h = C.c_void_p()
        raise_for_status(lib().gt_clone(self._h, device, C.byref(h)), _err())
        c = DeviceDag.__new__(DeviceDag)
        c._h, c._blob, c.device, c.grammar, c._info = h, self._blob, device, self.grammar, None
        return c

    def sum_word_counts(self, shards) -> None:
        """gt_sum_word_counts: the shards' dense word counts (after a word
        count run on each) summed on this context's device through peer
        memory; the total becomes this context's device word counts."""
        hs = (C.c_void_p * len(shards))(*[s._h.value for s in shards])
        raise_for_status(lib().gt_sum_word_counts(self._h, hs, len(shards)), _err())

    def sharded(self, workers: int, devices=None):
        """The corpus sharded by token-balanced file ranges over `workers`
        contexts (shard.ShardedDag); cached per worker count."""
        from .shard import ShardedDag
        cache = self.__dict__.setdefault("_sharded", {})
        key = (workers, tuple(devices) if devices else None)
        if key not in cache:
            cache[key] = ShardedDag(self, workers, devices)
        return cache[key]

    def dag_array(self, name: str) -> np.ndarray:
        L = lib()
        n = L.gt_dag_array(self._h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(f"{name}: {_err()}")
        out = np.zeros(max(n, 1), dtype=np.int64)
        L.gt_dag_array(self._h, name.encode(), out.ctypes.data, len(out))
        return out[:n]

    def profile(self, enable: bool) -> None:
        profile(enable, self._h)

    def profile_report(self) -> dict:
        """{kernel name: (launches, total_ms)} since the last report."""
        return profile_report(self._h)

    def flush_l2(self) -> None:
        raise_for_status(lib().gt_flush_l2(self._h), _err())

    def sync(self) -> None:
        raise_for_status(lib().gt_sync(self._h), _err())

    def close(self) -> None:
        for sd in self.__dict__.pop("_sharded", {}).values():
            sd.close()
        if self._h is not None:
            lib().gt_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def profile(enable: bool, handle=None) -> None:
    """Per-kernel CUDA-event timing on the calling thread (gt_profile); with
    no handle it can bracket a gt_open (DeviceDag construction)."""
    raise_for_status(lib().gt_profile(handle, 1 if enable else 0), _err())


def profile_report(handle=None) -> dict:
    """{kernel name: (launches, total_ms)} since the last report."""
    L = lib()
    n = L.gt_profile_report(handle, None, 0)
    buf = C.create_string_buffer(max(int(n), 1) + 16)
    L.gt_profile_report(handle, buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split("\t")
        out[name] = (int(cnt), float(ms))
    return out


def table_add_batch(keys, deltas, capacity: int, device: int = 0):
    """gt_table_add_batch: concurrent inserts into one device hash table;
    returns {key: count} of the occupied slots (raises ResourceError when full)."""
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    dl = np.ascontiguousarray(deltas, dtype=np.uint64)
    ok = np.empty(capacity, dtype=np.uint32)
    ov = np.empty(capacity, dtype=np.uint64)
    st = lib().gt_table_add_batch(device, k.ctypes.data, dl.ctypes.data, len(k), capacity,
                                  ok.ctypes.data, ov.ctypes.data)
    raise_for_status(st, _err())
    occ = ok != 0xFFFFFFFF
    return dict(zip(ok[occ].tolist(), ov[occ].tolist())), ok, ov


def gtdc_of(source) -> bytes | None:
    """GTDC bytes of a reference `Grammar` (grammar.py:30-72) or of a
    reference `Dag` (dag.py:32-52, via its `.grammar`), serialized as the
    reference's serialize_grammar (grammar.py:164-174) writes them; None for
    anything else.  Duck-typed: the reference package is not imported."""
    g = getattr(source, "grammar", source)
    d, bodies = getattr(g, "dictionary", None), getattr(g, "bodies", None)
    if d is None or bodies is None or not hasattr(d, "words") or not hasattr(d, "num_splitters"):
        return None
    from .corpus import serialize_bodies
    return serialize_bodies(list(d.words), int(d.num_splitters), list(bodies))


def build_dag(source, device: int = 0) -> DeviceDag:
    """GTDC bytes, a path to a .gtdc file, or the reference's own `Dag` /
    `Grammar` object (dag.py:32-52, grammar.py:30-72: its grammar is
    serialized and loaded) -> DeviceDag."""
    if isinstance(source, (str, Path)):
        source = Path(source).read_bytes()
    elif not isinstance(source, (bytes, bytearray, memoryview, tuple)):
        blob = gtdc_of(source)
        if blob is None:
            raise UsageError(f"build_dag: cannot load a {type(source).__name__}")
        source = blob
    return DeviceDag(source, device=device)


def as_device_dag(dag, device: int = 0):
    """The task entry points accept the reference's `Dag` too:
    a reference Dag / Grammar is loaded once and the DeviceDag cached on it;
    a DeviceDag (or any handle with `run`) passes through."""
    if hasattr(dag, "run"):
        return dag
    cached = getattr(dag, "_b200_device_dag", None)
    if cached is not None:
        return cached
    dd = build_dag(dag, device)
    try:
        setattr(dag, "_b200_device_dag", dd)
    except (AttributeError, TypeError):
        pass
    return dd
