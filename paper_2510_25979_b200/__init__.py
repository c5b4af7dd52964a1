"""B200-native AttnCache hot path (arXiv 2510.25979) — thin Python binding over libattncache.so.

The binding only marshals arguments: torch supplies device memory (``data_ptr``)
and streams (``cuda_stream``); every step of the path runs in the library's
CUDA kernels (include/attncache.h).  There is no CPU fallback: if the
extension is missing or the device is not sm_100a, calls raise.

Function names follow the C ABI (``attncache_search`` ...).  Paper mapping:
Alg. 1 VecDB.search + theta gate -> ``attncache_search``; Alg. 2 hit branch
``mat_mul(attn_map, v)`` -> ``attncache_apply_cached``; Alg. 2 miss branch
(softmax(QK^T/sqrt(d_k)) . V, Eq. 5) -> ``attncache_attend_full``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

__all__ = [
    "AttnCacheError", "Context", "Database", "lib_path", "load_library",
    "attncache_ctx_create", "attncache_ctx_destroy", "attncache_ctx_sync", "attncache_db_load",
    "attncache_db_free", "attncache_search", "attncache_search_keys", "attncache_keys_decode",
    "attncache_apply_cached", "attncache_attend_full", "attncache_route_plan", "attncache_gather_rows",
    "attncache_scatter_rows", "attncache_fetch_maps", "attncache_variant", "attncache_version", "attncache_launch_count",
    "attncache_packed_map_elems", "attncache_pack_maps", "pack_db_maps", "attncache_capture_maps", "attncache_rope",
    "attncache_affinity_plan", "attncache_project_features", "attncache_apply_cached_gqa", "attncache_attend_full_gqa",
    "attncache_capture_maps_gqa", "attncache_affinity_plan_device", "ABI_FUNCTIONS", "attncache_get_unique_id",
    "attncache_ctx_info", "attncache_set_batch_layout", "attncache_search_all", "attncache_apply_cached_local",
    "attncache_relocate_rows", "attncache_prefill_host", "attncache_linear", "attncache_ctx_set_sm_budget",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_PKG, "lib", "libattncache.so")

# every symbol include/attncache.h declares
ABI_FUNCTIONS = [
    "attncache_status_string", "attncache_last_error", "attncache_version", "attncache_ctx_create",
    "attncache_ctx_destroy", "attncache_ctx_sync", "attncache_db_load", "attncache_db_free", "attncache_search",
    "attncache_search_keys", "attncache_keys_decode", "attncache_apply_cached", "attncache_attend_full",
    "attncache_route_plan", "attncache_gather_rows", "attncache_scatter_rows", "attncache_fetch_maps",
    "attncache_variant", "attncache_launch_count", "attncache_packed_map_elems", "attncache_pack_maps",
    "attncache_capture_maps", "attncache_rope", "attncache_affinity_plan", "attncache_project_features",
    "attncache_apply_cached_gqa", "attncache_attend_full_gqa", "attncache_capture_maps_gqa",
    "attncache_affinity_plan_device", "attncache_get_unique_id", "attncache_ctx_info", "attncache_set_batch_layout",
    "attncache_search_all", "attncache_apply_cached_local", "attncache_relocate_rows", "attncache_prefill_host",
    "attncache_linear", "attncache_ctx_set_sm_budget",
]

_DT = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}


class _DbDesc(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("shard_begin", ctypes.c_int64), ("shard_count", ctypes.c_int64),
                ("feat_dim", ctypes.c_int32), ("feat_dtype", ctypes.c_int32), ("feats", ctypes.c_void_p),
                ("n_layers", ctypes.c_int32), ("n_heads", ctypes.c_int32), ("seq_len", ctypes.c_int32),
                ("map_dtype", ctypes.c_int32), ("maps", ctypes.c_void_p), ("map_layout", ctypes.c_int32),
                ("maps_noncausal", ctypes.c_int32)]


class AttnCacheError(RuntimeError):
    def __init__(self, status: int, name: str, detail: str):
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name


_lib = None


def load_library():
    """Loads libattncache.so (built in-tree by paper_2510_25979_b200.build). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise ImportError(f"libattncache.so not built at {lib_path}; run `python -m paper_2510_25979_b200.build` "
                          "(there is no CPU fallback)")
    if "ATTNCACHE_NCCL_LIB" not in os.environ:  # the NCCL copy torch uses (the library dlopens it on demand)
        try:
            import nvidia.nccl as _nv
            cand = os.path.join(list(_nv.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["ATTNCACHE_NCCL_LIB"] = cand
        except Exception:  # pragma: no cover - the system libnccl.so.2 is the fallback
            pass
    L = ctypes.CDLL(lib_path)
    P, I64, I32, F32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    sig = {
        "attncache_status_string": ([I32], ctypes.c_char_p),
        "attncache_last_error": ([], ctypes.c_char_p),
        "attncache_version": ([], I32),
        "attncache_launch_count": ([], ctypes.c_uint64),
        "attncache_variant": ([I32, I32, I32, I32], ctypes.c_char_p),
        "attncache_ctx_create": ([I32, I32, I32, P, ctypes.POINTER(P)], I32),
        "attncache_get_unique_id": ([P], I32),
        "attncache_ctx_info": ([P, P, P], I32),
        "attncache_ctx_set_sm_budget": ([P, I32, I32], I32),
        "attncache_set_batch_layout": ([P, P, I32], I32),
        "attncache_search_all": ([P, P, I64, F32, P, P, P, P], I32),
        "attncache_apply_cached_local": ([P, P, P, I64, I32, I32, I32, I32, I32, P, P, P], I32),
        "attncache_relocate_rows": ([P, P, I64, I64, P, P, P, P], I32),
        "attncache_linear": ([P, P, I64, I32, P, I32, I32, P, I32, I32, P, P], I32),
        "attncache_prefill_host": ([P, P, I64, F32, P, P, P, I32, I32, P, P, P, P, I32, I32], I32),
        "attncache_ctx_destroy": ([P], I32),
        "attncache_ctx_sync": ([P], I32),
        "attncache_db_load": ([P, ctypes.POINTER(_DbDesc), ctypes.POINTER(P)], I32),
        "attncache_db_free": ([P], I32),
        "attncache_search": ([P, P, I64, F32, P, P, P, P], I32),
        "attncache_search_keys": ([P, P, I64, P, P], I32),
        "attncache_keys_decode": ([P, I32, I64, F32, P, P, P, P], I32),
        "attncache_apply_cached": ([P, P, P, I64, I32, I32, I32, I32, P, P, P], I32),
        "attncache_attend_full": ([P, I64, I32, I32, I32, I32, I32, P, P, P, F32, P, P, P], I32),
        "attncache_route_plan": ([P, P, I64, P, I32, P, P, P, P], I32),
        "attncache_gather_rows": ([P, P, I64, I64, P, P], I32),
        "attncache_scatter_rows": ([P, P, I64, I64, P, P], I32),
        "attncache_fetch_maps": ([P, I64, I32, I32, P, P], I32),
        "attncache_packed_map_elems": ([I32], I64),
        "attncache_pack_maps": ([P, I64, I32, P, P], I32),
        "attncache_rope": ([P, I64, I32, I32, I32, F32, P], I32),
        "attncache_capture_maps": ([P, I64, I32, I32, I32, I32, I32, P, P, F32, P, I32, I32, P, P], I32),
        "attncache_affinity_plan": ([P, P, I64, P, I32, ctypes.c_double, ctypes.c_double, P, P], I32),
        "attncache_project_features": ([P, P, I64, I32, I32, P, P, I32, P, P, I32, I32, P, P], I32),
        "attncache_apply_cached_gqa": ([P, P, P, I64, I32, I32, I32, I32, I32, P, P, P], I32),
        "attncache_attend_full_gqa": ([P, I64, I32, I32, I32, I32, I32, I32, P, P, P, F32, P, P, P], I32),
        "attncache_capture_maps_gqa": ([P, I64, I32, I32, I32, I32, I32, I32, P, P, F32, P, I32, I32, P, P], I32),
        "attncache_affinity_plan_device": ([P, P, P, I64, P, I32, ctypes.c_double, ctypes.c_double, I32, P, P, P, P, P,
                                            P, P, P, P], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        L = load_library()
        raise AttnCacheError(status, L.attncache_status_string(status).decode(), L.attncache_last_error().decode())


def _p(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream, device) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")


class Context:
    """attncache_ctx: one per process and device.  rank/world/uid (a 128-byte attncache_get_unique_id from
    rank 0) make it COLLECTIVE: the library owns an NCCL communicator over the world's GPUs; world=1 with no
    uid is a local context.  ``Context.from_process_group`` creates one per rank of a torch.distributed
    group, using torch only to broadcast the uid."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, uid: Optional[bytes] = None):
        L = load_library()
        h = ctypes.c_void_p()
        ub = None
        if uid is not None:
            if len(uid) != 128:
                raise ValueError("uid must be the 128 bytes of attncache_get_unique_id")
            ub = ctypes.create_string_buffer(bytes(uid), 128)
        _check(L.attncache_ctx_create(int(device), int(rank), int(world), ub, ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        self.rank, self.world = int(rank), int(world)
        self.collective = uid is not None

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Context":
        """Every rank of `group` calls this: rank 0 makes the NCCL unique id, torch.distributed broadcasts its
        bytes (the only thing torch carries), and each rank creates its communicator-owning context."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [attncache_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls(device, rank, world, obj[0])

    def set_sm_budget(self, compute_sms: int, aux_sms: int):
        """CTA caps of the persistent layer kernels and of the search / placement / copy kernels (both default
        to the SM count); see attncache_ctx_set_sm_budget."""
        attncache_ctx_set_sm_budget(self, compute_sms, aux_sms)

    def set_batch_layout(self, home_counts):
        """Declares every rank's home batch size for the following collective calls (None clears it)."""
        attncache_set_batch_layout(self, home_counts)

    def sync(self):
        _check(load_library().attncache_ctx_sync(self.handle))

    def close(self):
        if self.handle:
            load_library().attncache_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class Database:
    """attncache_db: this rank's shard of the feature-vector DB and the attention-map DB
    ("Both databases share the same index").  Keeps the borrowed tensors alive.

    maps: DENSE [n][L][H][S][S] (packed=False) or PACKED [n][L][H][attncache_packed_map_elems(S)]
    (packed=True, seq_len required); see include/attncache.h attncache_map_layout."""

    def __init__(self, ctx: Context, feats: torch.Tensor, maps: Optional[torch.Tensor] = None,
                 n_global: Optional[int] = None, shard_begin: int = 0, packed: bool = False,
                 seq_len: Optional[int] = None, causal: bool = True):
        L = load_library()
        _dev(feats, "feats")
        S = 0
        if maps is not None:
            _dev(maps, "maps")
            if maps.shape[0] != feats.shape[0]:
                raise ValueError("maps and feats must hold the same entries")
            if packed:
                S = int(seq_len)
                if maps.dim() != 4 or maps.shape[3] != attncache_packed_map_elems(S):
                    raise ValueError("packed maps must be [n][L][H][attncache_packed_map_elems(S)]")
            else:
                if maps.dim() != 5 or maps.shape[3] != maps.shape[4]:
                    raise ValueError("dense maps must be [n][L][H][S][S]")
                S = maps.shape[3]
        n = feats.shape[0]
        desc = _DbDesc(n_global=n if n_global is None else int(n_global), shard_begin=int(shard_begin),
                       shard_count=n, feat_dim=feats.shape[1], feat_dtype=_DT[feats.dtype],
                       feats=feats.data_ptr() if n else None,
                       n_layers=maps.shape[1] if maps is not None else 0,
                       n_heads=maps.shape[2] if maps is not None else 0,
                       seq_len=S,
                       map_dtype=_DT[maps.dtype] if maps is not None else 0,
                       maps=maps.data_ptr() if (maps is not None and n) else None,
                       map_layout=1 if packed else 0, maps_noncausal=0 if causal else 1)
        h = ctypes.c_void_p()
        _check(L.attncache_db_load(ctx.handle, ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        self.ctx = ctx
        self.feats, self.maps = feats, maps
        self.packed, self.seq_len = packed, S
        self.n_layers = maps.shape[1] if maps is not None else 0
        self.n_heads = maps.shape[2] if maps is not None else 0
        self.n_global, self.shard_begin, self.shard_count = desc.n_global, desc.shard_begin, n
        self.device = feats.device

    def close(self):
        if self.handle:
            load_library().attncache_db_free(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


# ---- function-style API mirroring the C names ---------------------------------------------------

def attncache_version() -> int:
    return int(load_library().attncache_version())


def attncache_launch_count() -> int:
    """Kernels launched by the library so far in this process (for gpu_launches)."""
    return int(load_library().attncache_launch_count())


def attncache_variant(kind: str, dtype: torch.dtype, seq_len: int, head_dim: int) -> str:
    k = {"search": 0, "apply": 1, "attend": 2, "capture": 3, "project": 4}[kind]
    return load_library().attncache_variant(k, _DT[dtype], int(seq_len), int(head_dim)).decode()


def attncache_ctx_create(device: int = 0, rank: int = 0, world: int = 1, uid: Optional[bytes] = None) -> Context:
    return Context(device, rank, world, uid)


def attncache_get_unique_id() -> bytes:
    """128-byte NCCL unique id for a collective Context (rank 0 makes it; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().attncache_get_unique_id(buf))
    return buf.raw


def attncache_ctx_set_sm_budget(ctx: Context, compute_sms: int, aux_sms: int):
    _check(load_library().attncache_ctx_set_sm_budget(ctx.handle, int(compute_sms), int(aux_sms)))


def attncache_ctx_info(ctx: Context):
    r, w = ctypes.c_int32(), ctypes.c_int32()
    _check(load_library().attncache_ctx_info(ctx.handle, ctypes.byref(r), ctypes.byref(w)))
    return r.value, w.value


def attncache_set_batch_layout(ctx: Context, home_counts) -> None:
    if home_counts is None:
        _check(load_library().attncache_set_batch_layout(ctx.handle, None, 0))
        return
    import numpy as np
    hc = np.ascontiguousarray(list(home_counts), dtype=np.int64)
    _check(load_library().attncache_set_batch_layout(ctx.handle, ctypes.c_void_p(hc.ctypes.data), hc.shape[0]))


def attncache_ctx_destroy(ctx: Context) -> None:
    ctx.close()


def attncache_ctx_sync(ctx: Context) -> None:
    ctx.sync()


def attncache_db_load(ctx: Context, feats, maps=None, n_global=None, shard_begin=0) -> Database:
    return Database(ctx, feats, maps, n_global, shard_begin)


def attncache_db_free(db: Database) -> None:
    db.close()


def _vec(t: Optional[torch.Tensor], n: int, dtype, dev, what: str) -> torch.Tensor:
    """An output/input vector of n elements: allocated when None, else checked (dtype, length, device)."""
    if t is None:
        return torch.empty(n, dtype=dtype, device=dev)
    _dev(t, what)
    if t.dtype != dtype or t.dim() != 1 or t.shape[0] < n or t.device != dev:
        raise ValueError(f"{what} must be a contiguous {dtype} vector of >= {n} elements on {dev}")
    return t


def _mask(t: Optional[torch.Tensor], n: int, dev, what: str):
    """A uint8/bool row mask of n elements (None allowed)."""
    if t is None:
        return None
    _dev(t, what)
    if t.dtype not in (torch.uint8, torch.bool) or t.dim() != 1 or t.shape[0] != n or t.device != dev:
        raise ValueError(f"{what} must be a contiguous uint8/bool vector of {n} elements on {dev}")
    return t


def _check_queries(db: Database, queries: torch.Tensor):
    _dev(queries, "queries")
    if queries.dim() != 2 or queries.shape[1] != db.feats.shape[1] or queries.dtype != db.feats.dtype:
        raise ValueError(f"queries must be [B][{db.feats.shape[1]}] {db.feats.dtype} (the DB's feature dim and dtype; "
                         "no silent casts)")
    if queries.device != db.device:
        raise ValueError("queries must live on the database's device")


def attncache_search(db: Database, queries: torch.Tensor, tau: float, idx=None, score=None, hit=None, stream=None):
    """Alg. 1 l.255-257: returns (idx int64[B], score f32[B], hit u8[B]) of this rank's B home queries (on a
    collective Context: the global top-1 over every rank's shard)."""
    _check_queries(db, queries)
    B = queries.shape[0]
    dev = queries.device
    idx = _vec(idx, B, torch.int64, dev, "idx")
    score = _vec(score, B, torch.float32, dev, "score")
    hit = _vec(hit, B, torch.uint8, dev, "hit")
    _check(load_library().attncache_search(db.handle, _p(queries), B, float(tau), _p(idx), _p(score), _p(hit),
                                           _stream(stream, dev)))
    return idx, score, hit


def attncache_search_all(db: Database, queries: torch.Tensor, tau: float, total: Optional[int] = None, idx=None,
                         score=None, hit=None, stream=None):
    """The decisions of the WHOLE batch (every rank's home block in rank order) on every rank; `total` = the
    sum of the home batch sizes (the Context's batch layout, or this rank's B on a local Context)."""
    _check_queries(db, queries)
    B = queries.shape[0]
    dev = queries.device
    total = B if total is None else int(total)
    idx = _vec(idx, total, torch.int64, dev, "idx")
    score = _vec(score, total, torch.float32, dev, "score")
    hit = _vec(hit, total, torch.uint8, dev, "hit")
    _check(load_library().attncache_search_all(db.handle, _p(queries), B, float(tau), _p(idx), _p(score), _p(hit),
                                               _stream(stream, dev)))
    return idx, score, hit


def attncache_search_keys(db: Database, queries: torch.Tensor, keys=None, stream=None) -> torch.Tensor:
    """This shard's packed top-1 keys (int64 view of the u64 keys)."""
    _check_queries(db, queries)
    B = queries.shape[0]
    keys = _vec(keys, B, torch.int64, queries.device, "keys")
    _check(load_library().attncache_search_keys(db.handle, _p(queries), B, _p(keys), _stream(stream, queries.device)))
    return keys


def attncache_keys_decode(keys: torch.Tensor, tau: float, idx=None, score=None, hit=None, stream=None):
    """keys: [n_shards][B] (or [B]) packed keys -> cross-shard top-1 idx/score/hit."""
    _dev(keys, "keys")
    if keys.dtype != torch.int64:
        raise ValueError("keys must be int64 (the u64 bit patterns)")
    keys = keys.reshape(-1, keys.shape[-1])
    n_shards, B = keys.shape
    dev = keys.device
    idx = _vec(idx, B, torch.int64, dev, "idx")
    score = _vec(score, B, torch.float32, dev, "score")
    hit = _vec(hit, B, torch.uint8, dev, "hit")
    _check(load_library().attncache_keys_decode(_p(keys), n_shards, B, float(tau), _p(idx), _p(score), _p(hit),
                                                _stream(stream, dev)))
    return idx, score, hit


def _apply_args(db: Database, idx, V, O, hit, layer_begin, layer_end):
    _dev(V, "V")
    _dev(idx, "idx")
    layer_end = db.n_layers if layer_end is None else layer_end
    if idx.dtype != torch.int64 or idx.dim() != 1:
        raise ValueError("idx must be an int64 vector")
    if V.dim() != 5 or V.shape[0] != idx.shape[0]:
        raise ValueError("V must be [B][L'][Hkv][S][d] matching idx")
    H = db.n_heads if db.maps is not None else V.shape[2]
    want = (V.shape[0], V.shape[1], H, V.shape[3], V.shape[4])
    if O is None:
        O = torch.empty(want, dtype=V.dtype, device=V.device)
    _dev(O, "O")
    if tuple(O.shape) != want or O.dtype != V.dtype or O.device != V.device:
        raise ValueError("O must be [B][L'][H][S][d] with V's B, L', S, d, dtype and device")
    if idx.device != V.device:
        raise ValueError("idx must live on V's device")
    hit = _mask(hit, idx.shape[0], V.device, "hit")
    if db.maps is not None and (V.shape[1] != layer_end - layer_begin or V.shape[3] != db.seq_len):
        raise AttnCacheError(2, "ATTNCACHE_ERR_SHAPE", "V shape disagrees with the database (L', S)")
    return O, hit, layer_end


def attncache_apply_cached(db: Database, idx: torch.Tensor, V: torch.Tensor, O: Optional[torch.Tensor] = None,
                           hit: Optional[torch.Tensor] = None, layer_begin: int = 0, layer_end: Optional[int] = None,
                           stream=None) -> torch.Tensor:
    """Alg. 2 l.373-375: O[b] = maps[idx[b]] . V[b] for selected rows; V [B][L'][Hkv][S][d], O [B][L'][H][S][d]
    (Hkv = H: multi-head; Hkv < H dividing H: grouped-query attention, map head h reads V head h // (H // Hkv)).
    On a collective Context the hits are routed to the rank owning their entry and O comes back (COLLECTIVE)."""
    O, hit, layer_end = _apply_args(db, idx, V, O, hit, layer_begin, layer_end)
    _check(load_library().attncache_apply_cached_gqa(db.handle, _p(idx), _p(hit), V.shape[0], int(layer_begin),
                                                     int(layer_end), V.shape[4], V.shape[2], _DT[V.dtype], _p(V), _p(O),
                                                     _stream(stream, V.device)))
    return O


def attncache_apply_cached_local(db: Database, idx: torch.Tensor, V: torch.Tensor, O: Optional[torch.Tensor] = None,
                                 hit: Optional[torch.Tensor] = None, layer_begin: int = 0,
                                 layer_end: Optional[int] = None, stream=None) -> torch.Tensor:
    """The local A.V (rows whose entry lies in this shard; never communicates): the owner-affinity placement."""
    O, hit, layer_end = _apply_args(db, idx, V, O, hit, layer_begin, layer_end)
    _check(load_library().attncache_apply_cached_local(db.handle, _p(idx), _p(hit), V.shape[0], int(layer_begin),
                                                       int(layer_end), V.shape[4], V.shape[2], _DT[V.dtype], _p(V),
                                                       _p(O), _stream(stream, V.device)))
    return O


def attncache_apply_cached_gqa(db: Database, idx: torch.Tensor, V: torch.Tensor, O: Optional[torch.Tensor] = None,
                               hit: Optional[torch.Tensor] = None, layer_begin: int = 0,
                               layer_end: Optional[int] = None, stream=None) -> torch.Tensor:
    """Grouped-query A.V (the C call of the same name); the head counts come from V and the database."""
    return attncache_apply_cached(db, idx, V, O, hit, layer_begin, layer_end, stream)


def attncache_attend_full(ctx: Context, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                          O: Optional[torch.Tensor] = None, scale: float = 0.0, skip: Optional[torch.Tensor] = None,
                          stream=None) -> torch.Tensor:
    """Alg. 2 l.376-381 / Eq. 5: O = softmax(QK^T*scale, causal) . V; Q, K, V, O [B][L][H][S][d]."""
    for t, n in ((Q, "Q"), (K, "K"), (V, "V")):
        _dev(t, n)
    if Q.dim() != 5 or K.shape != V.shape or not (Q.dtype == K.dtype == V.dtype) or \
            (K.shape[0], K.shape[1], K.shape[3], K.shape[4]) != (Q.shape[0], Q.shape[1], Q.shape[3], Q.shape[4]):
        raise ValueError("Q [B][L][H][S][d] and K, V [B][L][Hkv][S][d] must share B, L, S, d and dtype")
    if not (Q.device == K.device == V.device):
        raise ValueError("Q, K, V must live on one device")
    O = torch.empty_like(Q) if O is None else O
    _dev(O, "O")
    if O.shape != Q.shape or O.dtype != Q.dtype or O.device != Q.device:
        raise ValueError("O must have Q's shape, dtype and device")
    skip = _mask(skip, Q.shape[0], Q.device, "skip")
    B, Lq, H, S, d = Q.shape
    _check(load_library().attncache_attend_full_gqa(ctx.handle, B, Lq, H, K.shape[2], S, d, _DT[Q.dtype], _p(Q), _p(K),
                                                    _p(V), float(scale), _p(skip), _p(O), _stream(stream, Q.device)))
    return O


def attncache_attend_full_gqa(ctx: Context, Q, K, V, O=None, scale: float = 0.0, skip=None, stream=None):
    """Grouped-query causal attention (the C call of the same name): K, V with Hkv heads."""
    return attncache_attend_full(ctx, Q, K, V, O, scale, skip, stream)


def attncache_prefill_host(db: Database, q: torch.Tensor, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                           tau: float, O: Optional[torch.Tensor] = None, idx=None, score=None, hit=None,
                           chunk: Optional[int] = None, depth: int = 4):
    """The whole single-rank step end to end from PINNED host tensors (include/attncache.h
    attncache_prefill_host): every copy happens inside the library call, which returns when O and
    idx/score/hit are in host memory.  q [B][D]; Q, K, V, O [B][L][H][S][d] (all layers of the DB).
    chunk None: rows per pipeline chunk chosen for ~192 MB of V per chunk, at most 16 (a smaller chunk shortens
    the ring's fill and drain: configs[2], 67 MB rows, 222 -> 209 ms per step from 16 to 2 rows;
    scripts/e2e_chunk_sweep.py)."""
    ts = [(q, "q"), (Q, "Q"), (K, "K"), (V, "V")]
    for t, nme in ts:
        if t.is_cuda or not t.is_pinned() or not t.is_contiguous():
            raise ValueError(f"{nme} must be a contiguous pinned host tensor")
    B = q.shape[0]
    if q.dim() != 2 or q.shape[1] != db.feats.shape[1] or q.dtype != db.feats.dtype:
        raise ValueError("q must be [B][D] in the DB's feature dim and dtype")
    if V.dim() != 5 or V.shape[0] != B or V.shape[1] != db.n_layers or V.shape[2] != db.n_heads or \
            V.shape[3] != db.seq_len or Q.shape != V.shape or K.shape != V.shape or not (Q.dtype == K.dtype == V.dtype):
        raise ValueError("Q, K, V must be [B][L][H][S][d] with the DB's L, H, S and one dtype")
    mk = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()  # noqa: E731
    O = mk(V.shape, V.dtype) if O is None else O
    idx = mk((B,), torch.int64) if idx is None else idx
    score = mk((B,), torch.float32) if score is None else score
    hit = mk((B,), torch.uint8) if hit is None else hit
    for t, nme, dt, shape in ((O, "O", V.dtype, V.shape), (idx, "idx", torch.int64, (B,)),
                              (score, "score", torch.float32, (B,)), (hit, "hit", torch.uint8, (B,))):
        if t.is_cuda or not t.is_pinned() or not t.is_contiguous() or t.dtype != dt or tuple(t.shape) != tuple(shape):
            raise ValueError(f"{nme} must be a contiguous pinned host {dt} tensor of shape {tuple(shape)}")
    if chunk is None:
        chunk = max(1, min(16, (192 << 20) // max(1, V[0].numel() * V.element_size())))
    _check(load_library().attncache_prefill_host(db.handle, _p(q), B, float(tau), _p(Q), _p(K), _p(V), V.shape[4],
                                                 _DT[V.dtype], _p(O), _p(idx), _p(score), _p(hit), int(chunk),
                                                 int(depth)))
    return idx, score, hit, O


def attncache_relocate_rows(ctx: Context, src: torch.Tensor, send_order: torch.Tensor, counts, dst=None, stream=None):
    """COLLECTIVE: moves this rank's home rows src[send_order] to the ranks the placement chose and returns
    the rows received from every rank, in rank order (include/attncache.h attncache_relocate_rows).  counts:
    the 2 world + 1 ints of attncache_affinity_plan_device (send_n | recv_n | n_loc; host sequence)."""
    import numpy as np
    _dev(src, "src")
    c = np.ascontiguousarray(list(counts), dtype=np.int32)
    w = (c.shape[0] - 1) // 2
    n_recv = int(c[w:2 * w].sum())
    row_shape = src.shape[1:]
    dst = torch.empty((n_recv, *row_shape), dtype=src.dtype, device=src.device) if dst is None else dst
    _dev(dst, "dst")
    n_home = src.shape[0]
    row_bytes = (src[0].numel() if n_home else int(np.prod(row_shape))) * src.element_size()
    so = send_order[:n_home].contiguous() if n_home else None
    _check(load_library().attncache_relocate_rows(ctx.handle, _p(src) if n_home else None, n_home, row_bytes, _p(so),
                                                  ctypes.c_void_p(c.ctypes.data), _p(dst) if n_recv else None,
                                                  _stream(stream, src.device)))
    return dst


def attncache_route_plan(idx, hit, shard_begins: torch.Tensor, owner=None, counts=None, order=None, stream=None):
    n = idx.shape[0]
    world = shard_begins.shape[0] - 1
    dev = idx.device
    owner = torch.empty(n, dtype=torch.int32, device=dev) if owner is None else owner
    counts = torch.empty(world, dtype=torch.int32, device=dev) if counts is None else counts
    order = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if order is None else order
    _check(load_library().attncache_route_plan(_p(idx), _p(hit), n, _p(shard_begins), world, _p(owner), _p(counts),
                                               _p(order), _stream(stream, dev)))
    return owner, counts, order


def attncache_gather_rows(src: torch.Tensor, rows: torch.Tensor, dst: Optional[torch.Tensor] = None, stream=None):
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 0
    dst = torch.empty((rows.shape[0], *src.shape[1:]), dtype=src.dtype, device=src.device) if dst is None else dst
    if rows.shape[0]:
        _check(load_library().attncache_gather_rows(_p(src), _p(rows), rows.shape[0], row_bytes, _p(dst),
                                                    _stream(stream, src.device)))
    return dst


def attncache_scatter_rows(src: torch.Tensor, rows: torch.Tensor, dst: torch.Tensor, stream=None):
    if rows.shape[0]:
        row_bytes = src[0].numel() * src.element_size()
        _check(load_library().attncache_scatter_rows(_p(src), _p(rows), rows.shape[0], row_bytes, _p(dst),
                                                     _stream(stream, src.device)))
    return dst


def attncache_fetch_maps(db: Database, idx: int, layer_begin: int = 0, layer_end: Optional[int] = None,
                         out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Literal AttnMapsDB.get(idx, n) (Alg. 1 l.259): DENSE [layers][H][S][S] maps of a local entry."""
    layer_end = db.n_layers if layer_end is None else layer_end
    S = db.seq_len
    out = torch.empty((layer_end - layer_begin, db.n_heads, S, S), dtype=db.maps.dtype,
                      device=db.maps.device) if out is None else out
    _check(load_library().attncache_fetch_maps(db.handle, int(idx), int(layer_begin), int(layer_end), _p(out),
                                               _stream(stream, db.maps.device)))
    return out


def attncache_packed_map_elems(seq_len: int) -> int:
    return int(load_library().attncache_packed_map_elems(int(seq_len)))


def attncache_pack_maps(dense: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """DENSE [..., S, S] maps -> PACKED [..., attncache_packed_map_elems(S)] (DB building, Fig. 4 step 3)."""
    _dev(dense, "dense")
    S = dense.shape[-1]
    if dense.shape[-2] != S or dense.element_size() != 2:
        raise ValueError("dense maps must be [..., S, S] 16-bit")
    P = attncache_packed_map_elems(S)
    out = torch.empty((*dense.shape[:-2], P), dtype=dense.dtype, device=dense.device) if out is None else out
    _dev(out, "out")
    n_maps = dense.numel() // (S * S)
    _check(load_library().attncache_pack_maps(_p(dense), n_maps, S, _p(out), _stream(stream, dense.device)))
    return out


def pack_db_maps(cfg_maps_fn, n_entries: int, L: int, H: int, S: int, dtype, device, chunk: int = 16) -> torch.Tensor:
    """Builds a PACKED map DB [n][L][H][P] by packing dense maps chunk by chunk; cfg_maps_fn(begin, out)
    fills a DENSE [count][L][H][S][S] staging buffer for entries [begin, begin + count)."""
    P = attncache_packed_map_elems(S)
    db = torch.empty((n_entries, L, H, P), dtype=dtype, device=device)
    stage = torch.empty((min(chunk, n_entries), L, H, S, S), dtype=dtype, device=device)
    for b in range(0, n_entries, chunk):
        cnt = min(chunk, n_entries - b)
        cfg_maps_fn(b, stage[:cnt])
        attncache_pack_maps(stage[:cnt], db[b:b + cnt])
    return db


def attncache_capture_maps(ctx: Context, Q: torch.Tensor, K: torch.Tensor, map_dtype=torch.bfloat16,
                           packed: bool = True, out: Optional[torch.Tensor] = None, scale: float = 0.0,
                           skip: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """DB building (Fig. 4 step 1): the causal softmax maps of Q, K as DB entries
    [B][L][H][map] (PACKED or DENSE [..][S][S]) in map_dtype."""
    for t, n in ((Q, "Q"), (K, "K")):
        _dev(t, n)
    if Q.dim() != 5 or K.dim() != 5 or Q.dtype != K.dtype or \
            (K.shape[0], K.shape[1], K.shape[3], K.shape[4]) != (Q.shape[0], Q.shape[1], Q.shape[3], Q.shape[4]):
        raise ValueError("Q [B][L][H][S][d] and K [B][L][Hkv][S][d] must share B, L, S, d and dtype")
    B, Lq, H, S, d = Q.shape
    if out is None:
        tail = (attncache_packed_map_elems(S),) if packed else (S, S)
        out = torch.empty((B, Lq, H, *tail), dtype=map_dtype, device=Q.device)
    _dev(out, "out")
    _check(load_library().attncache_capture_maps_gqa(ctx.handle, B, Lq, H, K.shape[2], S, d, _DT[Q.dtype], _p(Q), _p(K),
                                                     float(scale), _p(skip), _DT[out.dtype], 1 if packed else 0, _p(out),
                                                     _stream(stream, Q.device)))
    return out


def attncache_capture_maps_gqa(ctx: Context, Q, K, map_dtype=torch.bfloat16, packed: bool = True, out=None,
                               scale: float = 0.0, skip=None, stream=None):
    """Grouped-query capture (the C call of the same name): K with Hkv heads, one map per query head."""
    return attncache_capture_maps(ctx, Q, K, map_dtype, packed, out, scale, skip, stream)


def attncache_linear(ctx: Context, X: torch.Tensor, W: torch.Tensor, n_heads: int, bias=None, out=None,
                     stream=None) -> torch.Tensor:
    """f4 projection (Alg. 2 l.372, l.377-378): X [B][S][K] times W [N][K] (nn.Linear layout, N = n_heads * d),
    stored head-major as [B][1][n_heads][S][d] (one layer; the layout attend_full / apply_cached read)."""
    _dev(X, "X")
    _dev(W, "W")
    if X.dim() != 3 or W.dim() != 2 or W.shape[1] != X.shape[2] or X.dtype != W.dtype or W.shape[0] % n_heads:
        raise ValueError("linear: X [B][S][K], W [N][K] (one dtype), N a multiple of n_heads")
    B, S, K = X.shape
    N = W.shape[0]
    d = N // n_heads
    out = torch.empty(B, 1, n_heads, S, d, dtype=X.dtype, device=X.device) if out is None else out
    _dev(out, "out")
    if out.numel() != B * N * S or out.dtype != X.dtype:
        raise ValueError("linear: out must hold [B][n_heads][S][d] elements of X's dtype")
    if bias is not None:
        _dev(bias, "bias")
        if bias.dtype != torch.float32 or bias.shape != (N,):
            raise ValueError("linear: bias must be float32 [N]")
    _check(load_library().attncache_linear(ctx.handle, _p(X), B * S, K, _p(W), N, _DT[X.dtype], _p(bias), S, d,
                                           _p(out), _stream(stream, X.device)))
    return out


def attncache_rope(X: torch.Tensor, base: float = 10000.0, stream=None) -> torch.Tensor:
    """In-place RoPE (rotate-half) on X [..., S, d]; position = index along S (f4 block comparison)."""
    _dev(X, "X")
    S, d = X.shape[-2], X.shape[-1]
    _check(load_library().attncache_rope(_p(X), X.numel() // (S * d), S, d, _DT[X.dtype], float(base),
                                         _stream(stream, X.device)))
    return X


def attncache_affinity_plan_device(ctx: "Context", idx: torch.Tensor, hit: torch.Tensor, shard_begins, home_begins,
                                   rank: int, hit_cost: float = 1.0, miss_cost: float = 1.0, stream=None):
    """Owner-affinity placement on the device (include/attncache.h attncache_affinity_plan_device): the plan of
    attncache_affinity_plan, bitwise, plus this rank's relocation lists.  idx int64 / hit uint8 on the device
    ([n], the whole batch); shard_begins, home_begins: host sequences [world + 1].  Returns a dict of device
    tensors assign (int32 [n]), load (float64 [world]), loc / idx_loc (int64 [n]), hit_loc (uint8 [n]),
    send_order (int64 [home size]) and counts (int32 [2 world + 1] = send_n | recv_n | n_loc)."""
    import numpy as np
    _dev(idx, "idx")
    _dev(hit, "hit")
    sb = np.ascontiguousarray(list(shard_begins), dtype=np.int64)
    hb = np.ascontiguousarray(list(home_begins), dtype=np.int64)
    world = sb.shape[0] - 1
    n = idx.shape[0]
    if idx.dtype != torch.int64 or hit.dtype != torch.uint8 or hit.shape[0] != n:
        raise ValueError("affinity_plan_device: idx int64 [n], hit uint8 [n]")
    if hb.shape[0] != world + 1:
        raise ValueError("affinity_plan_device: home_begins must have world + 1 entries")
    dev = idx.device
    home = int(hb[rank + 1] - hb[rank]) if 0 <= rank < world else 0
    p = lambda t: ctypes.c_void_p(t.data_ptr()) if t.numel() else None  # noqa: E731
    st = torch.cuda.current_stream(dev) if stream is None else stream
    with torch.cuda.stream(st):  # the outputs (and the counts' zero fill) are ordered on the launch stream
        out = _plan_outputs(n, world, home, dev)
    _check(load_library().attncache_affinity_plan_device(
        ctx.handle, p(idx.contiguous()), p(hit.contiguous()), n, ctypes.c_void_p(sb.ctypes.data), world,
        float(hit_cost), float(miss_cost), int(rank), ctypes.c_void_p(hb.ctypes.data), p(out["assign"]),
        p(out["load"]), p(out["loc"]), p(out["idx_loc"]), p(out["hit_loc"]), p(out["send_order"]),
        p(out["counts"]), _stream(st, dev)))
    out["send_order"] = out["send_order"][:home]
    return out


def _plan_outputs(n, world, home, dev):
    return {"assign": torch.empty(n, dtype=torch.int32, device=dev),
           "load": torch.empty(max(world, 1), dtype=torch.float64, device=dev),
           "loc": torch.empty(n, dtype=torch.int64, device=dev), "idx_loc": torch.empty(n, dtype=torch.int64, device=dev),
           "hit_loc": torch.empty(n, dtype=torch.uint8, device=dev),
           "send_order": torch.empty(max(home, 1), dtype=torch.int64, device=dev),
           "counts": torch.zeros(2 * max(world, 1) + 1, dtype=torch.int32, device=dev)}


def attncache_affinity_plan(idx, hit, shard_begins, hit_cost: float = 1.0, miss_cost: float = 1.0):
    """Owner-affinity placement (host function): returns (assign int32[n], load float64[world]).
    idx/hit are torch tensors (any device; read on the host) or numpy arrays; the outputs follow the input
    kind (CPU torch tensors or numpy arrays)."""
    import numpy as np
    as_torch = isinstance(idx, torch.Tensor)
    if as_torch:
        idx = idx.detach().to("cpu", torch.int64).numpy()
        hit = hit.detach().to("cpu", torch.uint8).numpy()
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    hit = np.ascontiguousarray(hit, dtype=np.uint8)
    if isinstance(shard_begins, torch.Tensor):
        shard_begins = shard_begins.detach().cpu().numpy()
    sb = np.ascontiguousarray(shard_begins, dtype=np.int64)
    world = sb.shape[0] - 1
    n = idx.shape[0]
    assign = np.empty(n, dtype=np.int32)
    load = np.empty(max(world, 0), dtype=np.float64)
    ptr = lambda a: ctypes.c_void_p(a.ctypes.data) if a.size else None  # noqa: E731
    _check(load_library().attncache_affinity_plan(ptr(idx), ptr(hit), n, ptr(sb), world, float(hit_cost),
                                                  float(miss_cost), ptr(assign), ptr(load)))
    if as_torch:
        return torch.from_numpy(assign), torch.from_numpy(load)
    return assign, load


def attncache_project_features(ctx: Context, h: torch.Tensor, W1: torch.Tensor, b1: torch.Tensor, W2: torch.Tensor,
                               b2: torch.Tensor, feat_dtype=None, out: Optional[torch.Tensor] = None,
                               stream=None) -> torch.Tensor:
    """Alg. 1 l.254 feature_projector (f2): features = normalize(W2 relu(W1 h + b1) + b2) as [n][D] in feat_dtype
    (default: h's dtype).  h [n][E], W1 [Hd][E], W2 [D][Hd] (one dtype), b1 [Hd], b2 [D] fp32."""
    for t, nme in ((h, "h"), (W1, "W1"), (b1, "b1"), (W2, "W2"), (b2, "b2")):
        _dev(t, nme)
    if h.dim() != 2 or W1.dim() != 2 or W2.dim() != 2 or W1.shape[1] != h.shape[1] or W2.shape[1] != W1.shape[0]:
        raise ValueError("project_features: h [n][E], W1 [Hd][E], W2 [D][Hd]")
    if not (h.dtype == W1.dtype == W2.dtype) or b1.dtype != torch.float32 or b2.dtype != torch.float32:
        raise ValueError("project_features: h/W1/W2 share one dtype; b1/b2 are float32")
    if b1.shape != (W1.shape[0],) or b2.shape != (W2.shape[0],):
        raise ValueError("project_features: bias shapes")
    n, E = h.shape
    Hd, D = W1.shape[0], W2.shape[0]
    feat_dtype = h.dtype if feat_dtype is None else feat_dtype
    out = torch.empty((n, D), dtype=feat_dtype, device=h.device) if out is None else out
    _dev(out, "out")
    _check(load_library().attncache_project_features(ctx.handle, _p(h), n, E, _DT[h.dtype], _p(W1), _p(b1), Hd, _p(W2),
                                                     _p(b2), D, _DT[out.dtype], _p(out), _stream(stream, h.device)))
    return out
