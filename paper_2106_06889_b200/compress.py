"""Native compressor: text files -> GTDC bytes identical to the reference's
`gtadoc compress` (ingest.py + sequitur.py + serialize_grammar; cli.py:89-100),
through gt_compress (csrc/sequitur.cpp, host code: no GPU needed)."""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from .device import lib
from .errors import CorruptionError, IngestError, ResourceError, UsageError


def compress_files(files: list[tuple[str, bytes]]) -> tuple[bytes, dict]:
    """(name, raw bytes) pairs in corpus order -> (GTDC bytes, stats)."""
    if not files:
        raise UsageError("corpus must contain at least one file")
    names = [n for n, _ in files]
    if len(set(names)) != len(names):
        raise UsageError("file names must be unique")
    bufs = [bytes(b) for _, b in files]
    ptrs = (C.c_void_p * len(bufs))(*[C.cast(C.c_char_p(b), C.c_void_p) for b in bufs])
    lens = np.asarray([len(b) for b in bufs], dtype=np.uint64)
    out, n = C.c_void_p(), C.c_uint64()
    stats = np.zeros(4, dtype=np.uint64)
    L = lib()
    st = L.gt_compress(ptrs, lens.ctypes.data, len(bufs), C.byref(out), C.byref(n), stats.ctypes.data)
    if st != 0:
        msg = L.gt_compress_last_error().decode()
        if st == 101:  # ingest.py:30-42 message: "<name>: invalid UTF-8 at byte offset N"
            raise IngestError(f"{names[int(stats[0])]}: {msg.split(': ', 1)[1]}")
        raise {1: UsageError, 2: ResourceError}.get(st, CorruptionError)(msg)
    try:
        blob = C.string_at(out, n.value) if n.value < (1 << 31) else \
            bytes((C.c_char * n.value).from_address(out.value))
    finally:
        L.gt_compress_free(out)
    return blob, dict(files=int(stats[0]), rules=int(stats[1]), vocabulary=int(stats[2]),
                      symbols=int(stats[3]))


def compress_dir(input_dir) -> tuple[bytes, dict]:
    """cli.py:69-82 _ingest_dir: regular files in lexicographic name order."""
    root = Path(input_dir)
    if not root.is_dir():
        raise UsageError(f"{input_dir}: not a directory")
    names = sorted(p.name for p in root.iterdir() if p.is_file())
    if not names:
        raise UsageError(f"{input_dir}: contains no regular files")
    return compress_files([(name, (root / name).read_bytes()) for name in names])


def tokenize_files(files: list[tuple[str, bytes]]):
    """(name, raw bytes) pairs -> (u32 token ids, u64 file offsets [nfiles+1])
    with the ids gt_compress gives the same files (gt_tokenize)."""
    bufs = [bytes(b) for _, b in files]
    ptrs = (C.c_void_p * len(bufs))(*[C.cast(C.c_char_p(b), C.c_void_p) for b in bufs])
    lens = np.asarray([len(b) for b in bufs], dtype=np.uint64)
    off = np.zeros(len(bufs) + 1, dtype=np.uint64)
    out = C.c_void_p()
    L = lib()
    st = L.gt_tokenize(ptrs, lens.ctypes.data, len(bufs), C.byref(out), off.ctypes.data)
    if st != 0:
        raise {1: IngestError, 2: ResourceError}.get(st, UsageError)(L.gt_compress_last_error().decode())
    try:
        n = int(off[-1])
        toks = np.ctypeslib.as_array((C.c_uint32 * max(n, 1)).from_address(out.value))[:n].copy()
    finally:
        L.gt_compress_free(out)
    return toks, off


def read_dir(input_dir) -> list[tuple[str, bytes]]:
    """cli.py:69-82 _ingest_dir order: regular files, lexicographic names."""
    root = Path(input_dir)
    if not root.is_dir():
        raise UsageError(f"{input_dir}: not a directory")
    names = sorted(p.name for p in root.iterdir() if p.is_file())
    if not names:
        raise UsageError(f"{input_dir}: contains no regular files")
    return [(name, (root / name).read_bytes()) for name in names]

