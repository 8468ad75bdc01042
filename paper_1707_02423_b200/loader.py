"""Native corpus loader: listings and profiles straight
to transition matrices, without the Python parse.

The reference builds each kernel's matrix in Python
(``cli.py:55-74`` ``_load_kernel``: ``parse_listing`` → ``build_cfg`` →
``parse_profiles`` / ``attribute_profile`` → ``transition_matrix``, then
``cli.py:77-79`` sorts by kernel id).  Here one C-ABI call
(``cfgsim_matrices_from_listings``, host C++ in ``csrc/loader.cpp``,
multi-threaded over kernels) does all of it.  Entries and ordering are
identical to the reference's; errors are the reference's classes with the
same line numbers and messages (``ListingSyntaxError``, ``UnresolvedLabel``,
``ProfileSyntaxError``, ``DuplicateKernel``, ``EmptyGraph``, ``CorpusError``,
and the plain ``ValueError`` / ``IndexError`` that ``KernelProfile`` and
``parse_profiles`` let escape).
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Iterable
from pathlib import Path

import numpy as np

from . import _native as nat
from .errors import (CorpusError, DuplicateKernel, EmptyGraph, ListingSyntaxError, ProfileSyntaxError,
                     UnresolvedLabel)
from .matrix import GLOBAL, RAW_COUNTS, ROW_STOCHASTIC, TransitionMatrix

__all__ = ["KernelSource", "matrices_from_listings", "load_manifest", "load_corpus_matrices"]


class KernelSource(tuple):
    """(kernel_id, listing text, profile text or None) — one corpus entry's inputs."""

    def __new__(cls, kernel_id: str, listing: str, profile: str | None = None):
        return super().__new__(cls, (kernel_id, listing, profile))


def _raise(code: int, line_no: int, msg: str, profile_name: str | None):
    if code == nat.ERR_LISTING_SYNTAX:
        raise ListingSyntaxError(line_no, msg)
    if code == nat.ERR_PROFILE_SYNTAX:
        raise ProfileSyntaxError(line_no, msg)
    if code == nat.ERR_UNRESOLVED_LABEL:
        raise UnresolvedLabel(msg)
    if code == nat.ERR_DUPLICATE_KERNEL:
        raise DuplicateKernel(msg)
    if code == nat.ERR_EMPTY_GRAPH:
        raise EmptyGraph(msg)
    if code == nat.ERR_CORPUS:  # cli.py:63-66 names the profile file
        raise CorpusError(msg.replace("profile has", f"{profile_name} has", 1) if profile_name else msg)
    if code == nat.ERR_VALUE:
        raise ValueError(msg)
    if code == nat.ERR_INDEX:
        raise IndexError(msg)
    if code == nat.ERR_NOMEM:
        raise MemoryError(msg)
    raise ValueError(msg)


def matrices_from_listings(kernels: Iterable, mode: str = ROW_STOCHASTIC, *, threads: int = 0,
                           profile_names: list[str | None] | None = None,
                           _matrix_rank: list[int] | None = None) -> list[TransitionMatrix]:
    """Transition matrices of ``kernels`` — ``(kernel_id, listing_text,
    profile_text | None)`` triples — in input order; the first failing kernel
    (input order) raises the reference's exception for it."""
    if mode not in (ROW_STOCHASTIC, GLOBAL, RAW_COUNTS):
        raise ValueError(f"unknown mode {mode!r}")
    ks = [tuple(k) for k in kernels]
    count = len(ks)
    if count == 0:
        return []
    ids = [str(k[0]).encode() for k in ks]
    lst = [k[1].encode() if isinstance(k[1], str) else bytes(k[1]) for k in ks]
    prf = [None if len(k) < 3 or k[2] is None else (k[2].encode() if isinstance(k[2], str) else bytes(k[2]))
           for k in ks]
    c_ids = (C.c_char_p * count)(*ids)
    c_lst = (C.c_char_p * count)(*lst)
    c_llen = np.array([len(x) for x in lst], np.int64)
    c_prf = (C.c_char_p * count)(*prf)
    c_plen = np.array([0 if x is None else len(x) for x in prf], np.int64)
    handle = C.c_void_p()
    rc = nat.lib.cfgsim_matrices_from_listings(count, C.cast(c_ids, C.c_void_p), C.cast(c_lst, C.c_void_p),
                                               nat.ptr(c_llen), C.cast(c_prf, C.c_void_p), nat.ptr(c_plen),
                                               nat.MODE_IDS[mode], int(threads), C.byref(handle))
    if handle.value is None:
        nat.check(rc if rc != nat.OK else nat.ERR_ARG)
    try:
        if rc != nat.OK:
            code, line = np.zeros(1, np.int32), np.zeros(1, np.int64)
            buf = C.create_string_buffer(4096)
            # cli.py loads every kernel before building any matrix, so a load
            # error anywhere wins over an earlier kernel's EmptyGraph
            first = None
            for k in range(count):
                nat.lib.cfgsim_matrices_status(handle, k, nat.ptr(code), nat.ptr(line), buf, len(buf))
                c = int(code[0])
                if c == nat.OK:
                    continue
                err = (c, int(line[0]), buf.value.decode(errors="replace"),
                       profile_names[k] if profile_names else None)
                if c != nat.ERR_EMPTY_GRAPH:
                    _raise(*err)
                rank = _matrix_rank[k] if _matrix_rank else k  # the order matrices are built in
                if first is None or rank < first[0]:
                    first = (rank, err)
            _raise(*first[1])
        sizes = np.zeros(count, np.int32)
        total = np.zeros(1, np.int64)
        nat.check(nat.lib.cfgsim_matrices_sizes(handle, nat.ptr(sizes), nat.ptr(total)))
        entries = np.empty(int(total[0]), np.float64)
        order = np.empty(int(sizes.astype(np.int64).sum()), np.int32)
        nat.check(nat.lib.cfgsim_matrices_read(handle, nat.ptr(entries), nat.ptr(order)))
    finally:
        nat.lib.cfgsim_matrices_destroy(handle)
    out = []
    e = o = 0
    for k in range(count):
        n = int(sizes[k])
        out.append(TransitionMatrix(ks[k][0], entries[e:e + n * n].reshape(n, n),
                                    tuple(order[o:o + n].tolist()), mode))
        e += n * n
        o += n
    return out


def load_manifest(path: str | Path) -> list[tuple[str, Path, Path | None, str]]:
    """``corpus.py:32-79`` ``load_manifest``: (kernel_id, listing, profile, arch)
    per line, paths relative to the manifest, the reference's CorpusErrors."""
    path = Path(path)
    try:
        text = path.read_text()
    except OSError as exc:
        raise CorpusError(f"cannot read manifest {path}: {exc}") from exc
    root = path.parent
    entries, seen = [], set()
    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tokens = line.split()
        if len(tokens) == 3:
            kernel_id, listing, arch = tokens
            profile = None
        elif len(tokens) == 4:
            kernel_id, listing, profile, arch = tokens
        else:
            raise CorpusError(f"{path}:{line_no}: expected 3 or 4 fields, got {len(tokens)}")
        if kernel_id in seen:
            raise CorpusError(f"{path}:{line_no}: duplicate kernel_id {kernel_id!r}")
        seen.add(kernel_id)
        listing_path = root / listing
        if not listing_path.is_file():
            raise CorpusError(f"{path}:{line_no}: listing not readable: {listing_path}")
        profile_path = None
        if profile is not None:
            profile_path = root / profile
            if not profile_path.is_file():
                raise CorpusError(f"{path}:{line_no}: profile not readable: {profile_path}")
        entries.append((kernel_id, listing_path, profile_path, arch))
    return entries


def load_corpus_matrices(manifest: str | Path, mode: str = ROW_STOCHASTIC, *,
                         threads: int = 0) -> list[TransitionMatrix]:
    """``cli.py:77-79`` + ``cli.py:88-89``: every kernel of a manifest, sorted
    by kernel id, as transition matrices (the ISO path's input)."""
    entries = load_manifest(manifest)
    profile_text: dict[Path, str] = {}
    ks, names = [], []
    for kid, lpath, ppath, _arch in entries:
        if ppath is not None and ppath not in profile_text:
            profile_text[ppath] = ppath.read_text()
        ks.append((kid, lpath.read_text(), None if ppath is None else profile_text[ppath]))
        names.append(None if ppath is None else str(ppath))
    by_id = sorted(range(len(ks)), key=lambda k: ks[k][0])
    rank = [0] * len(ks)
    for r, k in enumerate(by_id):
        rank[k] = r
    mats = matrices_from_listings(ks, mode, threads=threads, profile_names=names, _matrix_rank=rank)
    return [mats[k] for k in by_id]
