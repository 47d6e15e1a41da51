"""ctypes binding of libsa (include/sa.h) -- argument marshalling only.

Every function here has the name of the C entry point it wraps and does no
arithmetic of the method: it checks dtypes / devices / contiguity, allocates
outputs as torch tensors (torch is used for device memory, streams and
torch.distributed only) and calls the library.  There is no CPU fallback: if
``libsa.so`` is missing or no CUDA device is usable the call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# SA_LIBSA: another in-tree build of the same library (A/B experiments, scripts/build_variant.sh)
LIB_PATH = os.environ.get("SA_LIBSA") or os.path.join(_PKG, "lib", "libsa.so")

SA_OK, SA_E_INVAL, SA_E_RANGE, SA_E_CUDA, SA_E_COMM, SA_E_NOMEM, SA_E_STATE = range(7)
STATUS_NAMES = {0: "SA_OK", 1: "SA_E_INVAL", 2: "SA_E_RANGE", 3: "SA_E_CUDA", 4: "SA_E_COMM",
                5: "SA_E_NOMEM", 6: "SA_E_STATE"}
PHASES = ["S2a", "S2b", "S2c", "S2d", "S3", "S5", "rank", "gemm", "gemm_S2a", "gemm_S2d", "gemm_S5"]
PHASE_RING = 64

EXPORTED = ["sa_ctx_create", "sa_ctx_attach_comm", "sa_ctx_destroy", "sa_last_error", "sa_launch_count",
            "sa_ctx_set_timing", "sa_ctx_phase_ms", "sa_profile_stride", "sa_kmer_profiles", "sa_kmer_rank",
            "sa_partition", "sa_redistribute", "sa_bucket_similarity", "sa_exact_rank_compare", "sa_ctx_engine",
            "sa_ctx_set_rank_form", "sa_ctx_tc_columns", "sa_ctx_tc_operand", "sa_selftest_f_division",
            "sa_bucket_similarity_batch", "sa_pack_upper_u16", "sa_pack_upper_f64", "sa_guide_tree",
            "sa_guide_tree_batch", "sa_ctx_set_tree_form", "sa_ctx_tree_uncertified",
            "sa_ctx_phase_history", "sa_ctx_tc_sparse", "sa_nccl_unique_id", "sa_ctx_attach_nccl", "sa_ctx_check"]
SA_RANK_F, SA_RANK_DF = 0, 1
SA_TREE_F, SA_TREE_DF = 0, 1


class SaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class sa_key128(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_uint64), ("hi", ctypes.c_uint64)]


class sa_pivot(ctypes.Structure):
    _fields_ = [("key", sa_key128), ("global_idx", ctypes.c_int64), ("nk", ctypes.c_int32), ("block", ctypes.c_int32)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_void_p)
ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p)


class sa_comm_ops(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("allgather", ALLGATHER_FN), ("alltoallv", ALLTOALLV_FN)]


class sa_partition_debug(ctypes.Structure):
    _fields_ = [("local_key", ctypes.c_void_p), ("local_f64", ctypes.c_void_p), ("local_order", ctypes.c_void_p),
                ("sample_idx", ctypes.c_void_p), ("global_key", ctypes.c_void_p), ("global_f64", ctypes.c_void_p),
                ("global_order", ctypes.c_void_p), ("candidates", ctypes.c_void_p),
                ("exact_fallbacks_h", ctypes.POINTER(ctypes.c_int32)),
                ("uncertified_h", ctypes.POINTER(ctypes.c_int32)), ("global_num", ctypes.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libsa.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libsa.so not found at {path}; run `python -m paper_0905_1744_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I32, I64, VP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "sa_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
        "sa_ctx_attach_comm": (ctypes.c_int, [P, ctypes.POINTER(sa_comm_ops), ctypes.c_int, ctypes.c_int]),
        "sa_ctx_destroy": (ctypes.c_int, [P]),
        "sa_last_error": (ctypes.c_char_p, []),
        "sa_launch_count": (I64, []),
        "sa_ctx_set_timing": (ctypes.c_int, [P, ctypes.c_int]),
        "sa_ctx_phase_ms": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_float)]),
        "sa_profile_stride": (I32, [I32]),
        "sa_kmer_profiles": (ctypes.c_int, [P, P, P, I32, I32, I32, P, P, VP]),
        "sa_kmer_rank": (ctypes.c_int, [P, P, P, I32, P, P, I32, I32, P, P, P, VP]),
        "sa_partition": (ctypes.c_int, [P, I32, I32, P, P, P, I32, I64, I64, I32, P, P,
                                        ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(sa_partition_debug), VP]),
        "sa_redistribute": (ctypes.c_int, [P, I32, P, P, I32, I64, P, ctypes.POINTER(ctypes.c_int64),
                                           ctypes.POINTER(ctypes.c_int64), P, P, P, P, VP]),
        "sa_bucket_similarity": (ctypes.c_int, [P, P, P, I32, I32, P, P, VP]),
        "sa_bucket_similarity_batch": (ctypes.c_int, [P, I32, P, P, ctypes.POINTER(ctypes.c_int64), I32,
                                                      ctypes.POINTER(ctypes.c_void_p),
                                                      ctypes.POINTER(ctypes.c_void_p),
                                                      ctypes.POINTER(ctypes.c_int64), VP]),
        "sa_exact_rank_compare": (ctypes.c_int, [P, I32, P, I32, P, I32]),
        "sa_pack_upper_u16": (ctypes.c_int, [P, P, I32, ctypes.c_int64, P, VP]),
        "sa_pack_upper_f64": (ctypes.c_int, [P, P, I32, ctypes.c_int64, P, VP]),
        "sa_ctx_phase_history": (ctypes.c_int32, [P, ctypes.c_int32, ctypes.POINTER(ctypes.c_float), ctypes.c_int32]),
        "sa_guide_tree": (ctypes.c_int, [P, P, I32, ctypes.c_int64, P, P, VP]),
        "sa_guide_tree_batch": (ctypes.c_int, [P, I32, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int32),
                                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p),
                                               ctypes.POINTER(ctypes.c_void_p), VP]),
        "sa_ctx_engine": (ctypes.c_int, [P]),
        "sa_ctx_tc_columns": (ctypes.c_int32, [P, P, ctypes.c_int32]),
        "sa_ctx_tc_operand": (ctypes.c_int, [P]),
        "sa_ctx_tc_sparse": (ctypes.c_int32, [P, P, P, ctypes.c_int32]),
        "sa_nccl_unique_id": (ctypes.c_int, [P]),
        "sa_ctx_attach_nccl": (ctypes.c_int, [P, P, ctypes.c_int, ctypes.c_int]),
        "sa_ctx_check": (ctypes.c_int, [P, VP]),
        "sa_selftest_f_division": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]),
        "sa_ctx_set_rank_form": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_double]),
        "sa_ctx_set_tree_form": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_double]),
        "sa_ctx_tree_uncertified": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int64), VP]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(status: int):
    if status != SA_OK:
        raise SaError(status, load_library().sa_last_error().decode(errors="replace"))


def _ptr(t):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _dev(t, dtype, name):
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor (libsa has no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return t


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def sa_profile_stride(bins: int) -> int:
    return int(load_library().sa_profile_stride(bins))


def sa_exact_rank_compare(Ca, nka: int, Cb, nkb: int, nk_pool) -> int:
    """Host-side exact sign of V_a - V_b (sa.h); numpy inputs."""
    Ca = np.ascontiguousarray(Ca, dtype=np.uint16)
    Cb = np.ascontiguousarray(Cb, dtype=np.uint16)
    nkp = np.ascontiguousarray(nk_pool, dtype=np.int32)
    return int(load_library().sa_exact_rank_compare(Ca.ctypes.data, nka, Cb.ctypes.data, nkb, nkp.ctypes.data,
                                                    nkp.shape[0]))


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through libsa (sa_nccl_unique_id): 128 bytes."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().sa_nccl_unique_id(buf))
    return buf.raw


def sa_launch_count() -> int:
    return int(load_library().sa_launch_count())


# ---------------------------------------------------------------- context --
class Context:
    """An ``sa_ctx`` bound to one CUDA device (one per process and GPU)."""

    def __init__(self, device: int | None = None):
        lib = load_library()
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        h = ctypes.c_void_p()
        _check(lib.sa_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.nranks, self.rank = 1, 0
        self._comm_keepalive = None

    def close(self):
        if self.handle:
            load_library().sa_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int):
        """libsa's own NCCL communicator (sa_ctx_attach_nccl; collective): every
        rank passes the same 128-byte id (nccl_unique_id() on one rank, shared
        by the caller, e.g. with torch.distributed.broadcast_object_list)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(load_library().sa_ctx_attach_nccl(self.handle, buf, nranks, rank))
        self.nranks, self.rank = nranks, rank

    def check(self, stream=None):
        """sa_ctx_check: synchronise the stream, raise the sticky device errors
        of the asynchronous calls (SA_E_RANGE) or an NCCL asynchronous error."""
        _check(load_library().sa_ctx_check(self.handle, _stream(stream)))

    def attach_comm(self, comm: "TorchComm"):
        ops = comm.ops()
        self._comm_keepalive = (comm, ops)
        _check(load_library().sa_ctx_attach_comm(self.handle, ctypes.byref(ops), comm.nranks, comm.rank))
        self.nranks, self.rank = comm.nranks, comm.rank

    def engine(self) -> str:
        """Operand encoding of the last min-sum launch ('u16', 'u8', 'u16imad')."""
        return {0: "u16", 1: "u8", 2: "u16imad", 4: "tc"}.get(int(load_library().sa_ctx_engine(self.handle)), "none")

    def tc_operand(self) -> str:
        """K2T operand format: 'e2m1' (kind::mxf4, default) or 'u8' (kind::i8); 'none' before any K2T call."""
        return {0: "u8", 1: "e2m1"}.get(int(load_library().sa_ctx_tc_operand(self.handle)), "none")

    def tc_columns(self) -> list[int]:
        """K2T only: kept threshold-layer columns K' of each problem of the last
        min-sum call ([] when a fallback engine ran)."""
        buf = (ctypes.c_int32 * 64)()
        n = int(load_library().sa_ctx_tc_columns(self.handle, ctypes.cast(buf, ctypes.c_void_p), 64))
        if n < 0:
            raise SaError(SA_E_CUDA, "sa_ctx_tc_columns failed")
        return list(buf[:n])

    def set_rank_form(self, form: int = SA_RANK_F, delta: float = 0.02):
        """SA_RANK_F (mean F, exact) or SA_RANK_DF (mean -ln(Delta + F), Eq. 2-3)."""
        _check(load_library().sa_ctx_set_rank_form(self.handle, int(form), float(delta)))

    def set_tree_form(self, form: int = SA_TREE_F, delta: float = 0.02):
        """N4's distance: SA_TREE_F (d = 1 - F) or SA_TREE_DF (d = CR(-ln(Delta + F)), Eq. 2)."""
        _check(load_library().sa_ctx_set_tree_form(self.handle, int(form), float(delta)))

    def tree_uncertified(self, stream=None) -> int:
        """Uncertified correctly-rounded logs of the last tree call (blocks)."""
        v = ctypes.c_int64(0)
        _check(load_library().sa_ctx_tree_uncertified(self.handle, ctypes.byref(v), _stream(stream)))
        return int(v.value)

    def tc_sparse(self) -> list[tuple[int, int]]:
        """(mode, correction terms) of each problem of the last K2T call:
        mode 1 = layers >= 2 as sparse epilogue corrections, 0 = as MMA columns."""
        mode = np.zeros(64, dtype=np.int32)
        terms = np.zeros(64, dtype=np.int64)
        n = int(load_library().sa_ctx_tc_sparse(self.handle, mode.ctypes.data, terms.ctypes.data, 64))
        if n < 0:
            raise SaError(SA_E_CUDA, "sa_ctx_tc_sparse failed")
        return [(int(mode[i]), int(terms[i])) for i in range(n)]

    def set_timing(self, enable: bool = True):
        _check(load_library().sa_ctx_set_timing(self.handle, int(enable)))

    def phase_ms(self) -> dict:
        arr = (ctypes.c_float * len(PHASES))()
        _check(load_library().sa_ctx_phase_ms(self.handle, arr))
        return {k: float(arr[i]) for i, k in enumerate(PHASES)}

    def phase_history(self, phase: str) -> list[float]:
        """Durations (ms) of the kept occurrences of one phase, oldest first
        (sa_ctx_phase_history; host-blocking -- call outside timed regions)."""
        arr = (ctypes.c_float * PHASE_RING)()
        n = int(load_library().sa_ctx_phase_history(self.handle, PHASES.index(phase), arr, PHASE_RING))
        if n < 0:
            raise SaError(SA_E_CUDA, "sa_ctx_phase_history failed")
        return [float(arr[i]) for i in range(n)]


# ------------------------------------------------------------- S1 .. S5 ----
def sa_kmer_profiles(ctx: Context, residues: torch.Tensor, offsets: torch.Tensor, k: int = 3, alphabet: int = 20,
                     profiles: torch.Tensor | None = None, nkmers: torch.Tensor | None = None, stream=None,
                     check: bool = False):
    """S1: returns (profiles uint16 [n][stride], nkmers int32 [n]) (sa.h).
    Asynchronous: range errors surface at ctx.check() (check=True calls it
    here) or at sa_partition's count exchange."""
    _dev(residues, torch.uint8, "residues")
    _dev(offsets, torch.int64, "offsets")
    n = offsets.numel() - 1
    bins = alphabet ** k
    stride = sa_profile_stride(bins) if bins <= 65536 else bins
    dev = offsets.device
    if profiles is None:
        profiles = torch.empty((max(n, 0), stride), dtype=torch.uint16, device=dev)
    if nkmers is None:
        nkmers = torch.empty(max(n, 0), dtype=torch.int32, device=dev)
    _check(load_library().sa_kmer_profiles(ctx.handle, _ptr(residues), _ptr(offsets), n, k, alphabet,
                                           _ptr(profiles), _ptr(nkmers), _stream(stream)))
    if check:
        ctx.check(stream)
    return profiles, nkmers


def selftest_f_division(device: int = 0) -> int:
    """Mismatches of the K2T epilogue's division-free F = C/D against IEEE RN
    division over every 0 <= C <= D <= 65535 (expected 0)."""
    n = ctypes.c_int64(-1)
    _check(load_library().sa_selftest_f_division(device, ctypes.byref(n)))
    return int(n.value)


def sa_kmer_rank(ctx: Context, q_prof, q_nk, pool_prof, pool_nk, bins: int = 8000, want_f64: bool = True,
                 want_numerators: bool = False, stream=None):
    """S2: returns (keys int64 [nq][2] as (lo, hi) bit patterns, rank_f64 | None, numerators | None)."""
    for t, name in ((q_prof, "q_prof"), (pool_prof, "pool_prof")):
        _dev(t, torch.uint16, name)
    _dev(q_nk, torch.int32, "q_nk")
    _dev(pool_nk, torch.int32, "pool_nk")
    nq, npool = q_nk.numel(), pool_nk.numel()
    dev = q_nk.device
    keys = torch.empty((nq, 2), dtype=torch.int64, device=dev)
    f64 = torch.empty(nq, dtype=torch.float64, device=dev) if want_f64 else None
    num = torch.empty((nq, npool), dtype=torch.uint16, device=dev) if want_numerators else None
    _check(load_library().sa_kmer_rank(ctx.handle, _ptr(q_prof), _ptr(q_nk), nq, _ptr(pool_prof), _ptr(pool_nk),
                                       npool, bins, _ptr(keys), _ptr(f64), _ptr(num), _stream(stream)))
    return keys, f64, num


@dataclass
class PartitionOut:
    bucket_of: torch.Tensor        # int32 [n_local]
    pivots: torch.Tensor           # int64 [p-1][4] raw sa_pivot records
    counts: np.ndarray             # int64 [nranks][p]
    bytes: np.ndarray              # int64 [nranks][p]
    debug: dict | None = None
    exact_fallbacks: int = 0
    uncertified: int = 0


def pivot_global_idx(pivots: torch.Tensor) -> torch.Tensor:
    return pivots[:, 2]


def sa_partition(ctx: Context, p: int, samples_per_block: int, profiles, nkmers, offsets, bins: int,
                 n_total: int, first_global: int, debug: bool = False, stream=None,
                 want_global_num: bool = False) -> PartitionOut:
    """S2a-S3c (Algorithm 2 steps 2-11) on this rank's shard; see sa.h."""
    _dev(profiles, torch.uint16, "profiles")
    _dev(nkmers, torch.int32, "nkmers")
    _dev(offsets, torch.int64, "offsets")
    n_local = nkmers.numel()
    dev = nkmers.device
    bucket_of = torch.empty(n_local, dtype=torch.int32, device=dev)
    pivots = torch.zeros((max(p - 1, 1), 4), dtype=torch.int64, device=dev)   # 32-byte sa_pivot records
    counts = np.zeros((ctx.nranks, p), dtype=np.int64)
    nbytes = np.zeros((ctx.nranks, p), dtype=np.int64)
    dbg_struct = None
    dbg = None
    fallbacks = ctypes.c_int32(0)
    uncertified = ctypes.c_int32(0)
    if debug:
        s = p * samples_per_block
        dbg = {
            "local_key": torch.empty((n_local, 2), dtype=torch.int64, device=dev),
            "local_f64": torch.empty(n_local, dtype=torch.float64, device=dev),
            "local_order": torch.empty(n_local, dtype=torch.int64, device=dev),
            "sample_idx": torch.empty(s, dtype=torch.int64, device=dev),
            "global_key": torch.empty((n_local, 2), dtype=torch.int64, device=dev),
            "global_f64": torch.empty(n_local, dtype=torch.float64, device=dev),
            "global_order": torch.empty(n_local, dtype=torch.int64, device=dev),
            "candidates": torch.empty(max(p * (p - 1), 1), dtype=torch.int64, device=dev),
        }
        if want_global_num:   # the S2d numerator matrix [n_local][s] (parity artifact)
            dbg["global_num"] = torch.empty((n_local, s), dtype=torch.uint16, device=dev)
        dbg_struct = sa_partition_debug(*[_ptr(dbg[k]) for k in ["local_key", "local_f64", "local_order",
                                                                  "sample_idx", "global_key", "global_f64",
                                                                  "global_order", "candidates"]],
                                        ctypes.pointer(fallbacks), ctypes.pointer(uncertified),
                                        _ptr(dbg.get("global_num")))
    _check(load_library().sa_partition(
        ctx.handle, p, samples_per_block, _ptr(profiles), _ptr(nkmers), _ptr(offsets), bins, n_total, first_global,
        n_local, _ptr(bucket_of), _ptr(pivots),
        counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), nbytes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        ctypes.byref(dbg_struct) if dbg_struct is not None else None, _stream(stream)))
    if dbg is not None:
        dbg["candidates"] = dbg["candidates"][:p * (p - 1)]
    return PartitionOut(bucket_of, pivots[:max(p - 1, 0)], counts, nbytes, dbg, int(fallbacks.value),
                        int(uncertified.value))


def owned_buckets(p: int, nranks: int, rank: int) -> range:
    """Buckets [rank*p/nranks, (rank+1)*p/nranks) live on `rank` (sa.h)."""
    pb = p // nranks
    return range(rank * pb, (rank + 1) * pb)


def recv_sizes(counts: np.ndarray, nbytes: np.ndarray, p: int, nranks: int, rank: int):
    """Receive-buffer sizes for sa_redistribute: (sequences, residue bytes)."""
    own = list(owned_buckets(p, nranks, rank))
    return int(counts[:, own].sum()), int(nbytes[:, own].sum())


def sa_redistribute(ctx: Context, p: int, residues, offsets, first_global: int, part: PartitionOut, stream=None):
    """S4: returns (recv_residues, recv_offsets, recv_global_idx, recv_bucket) ordered by (bucket, global id)."""
    _dev(residues, torch.uint8, "residues")
    _dev(offsets, torch.int64, "offsets")
    n_local = offsets.numel() - 1
    dev = offsets.device
    nseq, nres = recv_sizes(part.counts, part.bytes, p, ctx.nranks, ctx.rank)
    rres = torch.empty(max(nres, 1), dtype=torch.uint8, device=dev)
    roffs = torch.empty(nseq + 1, dtype=torch.int64, device=dev)
    rgid = torch.empty(max(nseq, 1), dtype=torch.int64, device=dev)
    rbkt = torch.empty(max(nseq, 1), dtype=torch.int32, device=dev)
    counts = np.ascontiguousarray(part.counts, dtype=np.int64)
    nbytes = np.ascontiguousarray(part.bytes, dtype=np.int64)
    _check(load_library().sa_redistribute(
        ctx.handle, p, _ptr(residues), _ptr(offsets), n_local, first_global, _ptr(part.bucket_of),
        counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), nbytes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        _ptr(rres), _ptr(roffs), _ptr(rgid), _ptr(rbkt), _stream(stream)))
    return rres[:nres], roffs, rgid[:nseq], rbkt[:nseq]


def sa_bucket_similarity(ctx: Context, profiles, nkmers, bins: int = 8000, want_numerators: bool = True,
                         want_similarity: bool = True, numerators=None, similarity=None, stream=None):
    """S5: returns (numerators uint16 [n][n] | None, similarity f64 [n][n] | None)."""
    _dev(profiles, torch.uint16, "profiles")
    _dev(nkmers, torch.int32, "nkmers")
    n = nkmers.numel()
    dev = nkmers.device
    if want_numerators and numerators is None:
        numerators = torch.empty((n, n), dtype=torch.uint16, device=dev)
    if want_similarity and similarity is None:
        similarity = torch.empty((n, n), dtype=torch.float64, device=dev)
    _check(load_library().sa_bucket_similarity(ctx.handle, _ptr(profiles), _ptr(nkmers), n, bins,
                                               _ptr(numerators), _ptr(similarity), _stream(stream)))
    return numerators, similarity


def padded_matrix(n: int, dtype, device, ld_align: int = 1):
    """An n x n view (row stride ld = n rounded up to ld_align) of an n x ld
    allocation: the padded layout sa_bucket_similarity_batch writes when
    given ld (whole 32-byte store sectors for ld_align = 16)."""
    ld = -(-n // ld_align) * ld_align
    return torch.empty((n, ld), dtype=dtype, device=device)[:, :n]


def _row_stride(t, n):
    if t is None:
        return None
    if t.dim() != 2 or t.shape[0] != n or t.shape[1] != n or t.stride(1) != 1 or t.stride(0) < n:
        raise ValueError("bucket matrix must be n x n with unit column stride")
    return t.stride(0)


def sa_bucket_similarity_batch(ctx: Context, profiles, nkmers, row_begin, bins: int = 8000,
                               want_numerators: bool = True, want_similarity: bool = True,
                               numerators=None, similarity=None, stream=None, ld_align: int = 1):
    """S5 over several buckets in one call: bucket b = rows [row_begin[b],
    row_begin[b+1]).  Returns (list of numerators | None, list of similarity | None),
    one entry per bucket (None for empty buckets or when not wanted).  Given or
    allocated matrices may be padded n x n views (row stride >= n, see
    padded_matrix; both of a bucket must share the stride)."""
    _dev(profiles, torch.uint16, "profiles")
    _dev(nkmers, torch.int32, "nkmers")
    nb = len(row_begin) - 1
    dev = nkmers.device
    sizes = [int(row_begin[b + 1]) - int(row_begin[b]) for b in range(nb)]
    if numerators is None:
        numerators = [padded_matrix(n, torch.uint16, dev, ld_align) if want_numerators and n else None
                      for n in sizes]
    if similarity is None:
        similarity = [padded_matrix(n, torch.float64, dev, ld_align) if want_similarity and n else None
                      for n in sizes]
    lds = []
    for n, t_num, t_sim in zip(sizes, numerators, similarity):
        a, b_ = _row_stride(t_num, n), _row_stride(t_sim, n)
        if a is not None and b_ is not None and a != b_:
            raise ValueError("numerators and similarity of a bucket must share the row stride")
        lds.append(a if a is not None else (b_ if b_ is not None else n))
    rb = (ctypes.c_int64 * (nb + 1))(*[int(x) for x in row_begin])
    ldh = (ctypes.c_int64 * max(nb, 1))(*lds)
    nums = (ctypes.c_void_p * max(nb, 1))(*[(t.data_ptr() if t is not None else None) for t in numerators])
    sims = (ctypes.c_void_p * max(nb, 1))(*[(t.data_ptr() if t is not None else None) for t in similarity])
    _check(load_library().sa_bucket_similarity_batch(ctx.handle, nb, _ptr(profiles), _ptr(nkmers), rb, bins,
                                                     nums, sims, ldh, _stream(stream)))
    return numerators, similarity


def sa_guide_tree(ctx: Context, similarity: torch.Tensor, stream=None):
    """N4: UPGMA guide tree of a bucket's similarity matrix (n x n fp64 view,
    any row stride >= n).  Returns (merges int32 [n-1][2], heights f64 [n-1])
    on the device (sa.h)."""
    if similarity.dtype != torch.float64 or not similarity.is_cuda or similarity.dim() != 2 \
            or similarity.shape[0] != similarity.shape[1] or similarity.stride(1) != 1:
        raise ValueError("similarity must be an n x n float64 CUDA tensor with contiguous rows")
    n = similarity.shape[0]
    merges = torch.empty((max(n - 1, 0), 2), dtype=torch.int32, device=similarity.device)
    heights = torch.empty(max(n - 1, 0), dtype=torch.float64, device=similarity.device)
    _check(load_library().sa_guide_tree(ctx.handle, ctypes.c_void_p(similarity.data_ptr()), n, similarity.stride(0),
                                        _ptr(merges), _ptr(heights), _stream(stream)))
    return merges, heights


def sa_guide_tree_batch(ctx: Context, similarities, stream=None):
    """N4 for several buckets in one launch (sa.h sa_guide_tree_batch): a list
    of n x n fp64 CUDA views; returns [(merges, heights)] in the same order."""
    sims = list(similarities)
    for t in sims:
        if t.dtype != torch.float64 or not t.is_cuda or t.dim() != 2 or t.shape[0] != t.shape[1] \
                or t.stride(1) != 1:
            raise ValueError("similarity must be an n x n float64 CUDA tensor with contiguous rows")
    k = len(sims)
    outs = []
    for t in sims:
        n = t.shape[0]
        outs.append((torch.empty((max(n - 1, 0), 2), dtype=torch.int32, device=t.device),
                     torch.empty(max(n - 1, 0), dtype=torch.float64, device=t.device)))
    arr = lambda xs: (ctypes.c_void_p * max(k, 1))(*xs)  # noqa: E731
    ns = (ctypes.c_int32 * max(k, 1))(*[t.shape[0] for t in sims])
    lds = (ctypes.c_int64 * max(k, 1))(*[t.stride(0) for t in sims])
    _check(load_library().sa_guide_tree_batch(ctx.handle, k, arr([t.data_ptr() for t in sims]), ns, lds,
                                              arr([m.data_ptr() for m, _ in outs]),
                                              arr([h.data_ptr() for _, h in outs]), _stream(stream)))
    return outs


def _pack_upper(fn: str, dtype, ctx: Context, matrix: torch.Tensor, packed: torch.Tensor | None, stream):
    if matrix.dtype != dtype or not matrix.is_cuda or matrix.dim() != 2 or matrix.shape[0] != matrix.shape[1]:
        raise ValueError(f"matrix must be an n x n {dtype} CUDA tensor")
    if matrix.stride(1) != 1:
        raise ValueError("matrix rows must be contiguous")
    n = matrix.shape[0]
    if packed is None:
        packed = torch.empty(n * (n + 1) // 2, dtype=dtype, device=matrix.device)
    _check(getattr(load_library(), fn)(ctx.handle, ctypes.c_void_p(matrix.data_ptr()), n, matrix.stride(0),
                                       _ptr(packed), _stream(stream)))
    return packed


def sa_pack_upper_u16(ctx: Context, matrix: torch.Tensor, packed: torch.Tensor | None = None, stream=None):
    """Packed upper triangle (diagonal included) of a symmetric n x n uint16
    matrix (n x n view with any row stride >= n): row i's columns i..n-1 at
    i*n - i*(i-1)/2; returns the n(n+1)/2 uint16 device tensor (sa.h)."""
    return _pack_upper("sa_pack_upper_u16", torch.uint16, ctx, matrix, packed, stream)


def sa_pack_upper_f64(ctx: Context, matrix: torch.Tensor, packed: torch.Tensor | None = None, stream=None):
    """The same for a symmetric fp64 similarity matrix (sa.h)."""
    return _pack_upper("sa_pack_upper_f64", torch.float64, ctx, matrix, packed, stream)


# ------------------------------------------------------- communicator -----
class _ArrayView:
    """Expose a raw device pointer to torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def raw_tensor(ptr: int, nbytes: int, device) -> torch.Tensor:
    """uint8 tensor aliasing `nbytes` at `ptr` (device memory, or host memory for CPU tests)."""
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    if torch.device(device).type == "cuda":
        return torch.as_tensor(_ArrayView(ptr, nbytes), device=device)
    buf = (ctypes.c_uint8 * nbytes).from_address(ptr)
    return torch.from_numpy(np.ctypeslib.as_array(buf))


class TorchComm:
    """sa_comm_ops implemented with torch.distributed (NCCL on GPUs; gloo with
    host buffers in the CPU tests).  Plumbing only: allgather and a variable
    all-to-all of bytes, ordered on the caller's stream."""

    def __init__(self, group=None, device="cuda", stage_host: bool = False):
        """stage_host: the buffers are device memory but the process group's
        backend is host-only (gloo): each collective copies through host
        memory (the multi-process test on one GPU, tests/test_gpu_two_process.py)."""
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device(device)
        self.stage_host = stage_host
        self.errors = []

    def _with_stream(self, stream_ptr):
        if self.device.type == "cuda" and stream_ptr:
            return torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr, device=self.device))
        import contextlib
        return contextlib.nullcontext()

    def allgather(self, user, send, recv, nbytes, stream):
        try:
            if self.stage_host:
                with self._with_stream(stream):
                    src = raw_tensor(send, nbytes, self.device).cpu()
                    parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.nranks)]
                    self.dist.all_gather(parts, src, group=self.group)
                    raw_tensor(recv, nbytes * self.nranks, self.device).copy_(torch.cat(parts))
                return 0
            with self._with_stream(stream):
                src = raw_tensor(send, nbytes, self.device)
                dst = raw_tensor(recv, nbytes * self.nranks, self.device)
                if send == recv:
                    src = src.clone()
                self.dist.all_gather_into_tensor(dst, src, group=self.group)
            return 0
        except Exception as e:  # errors cannot cross the C ABI as exceptions
            self.errors.append(repr(e))
            return 1

    def alltoallv(self, user, send, sbytes, sdispl, recv, rbytes, rdispl, stream):
        try:
            n = self.nranks
            sb = [int(sbytes[i]) for i in range(n)]
            rb = [int(rbytes[i]) for i in range(n)]
            sd = [int(sdispl[i]) for i in range(n)]
            rd = [int(rdispl[i]) for i in range(n)]
            assert sd == list(np.cumsum([0] + sb[:-1])) and rd == list(np.cumsum([0] + rb[:-1])), \
                "displacements must be packed prefix sums"
            with self._with_stream(stream):
                src = raw_tensor(send, sum(sb), self.device)
                dst = raw_tensor(recv, sum(rb), self.device)
                if self.stage_host:
                    hd = torch.empty(sum(rb), dtype=torch.uint8)
                    self.dist.all_to_all_single(hd, src.cpu(), output_split_sizes=rb, input_split_sizes=sb,
                                                group=self.group)
                    dst.copy_(hd)
                else:
                    self.dist.all_to_all_single(dst, src, output_split_sizes=rb, input_split_sizes=sb,
                                                group=self.group)
            return 0
        except Exception as e:
            self.errors.append(repr(e))
            return 1

    def ops(self) -> sa_comm_ops:
        self._ag = ALLGATHER_FN(self.allgather)
        self._a2a = ALLTOALLV_FN(self.alltoallv)
        return sa_comm_ops(None, self._ag, self._a2a)


def keys_to_ints(keys: torch.Tensor) -> list:
    """int64 [n][2] (lo, hi) bit patterns -> Python ints (128-bit keys)."""
    k = keys.detach().cpu().numpy().view(np.uint64)
    return [int(lo) | (int(hi) << 64) for lo, hi in k]
