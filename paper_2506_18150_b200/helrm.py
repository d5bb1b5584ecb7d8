"""Thin ctypes binding of libhelrm.so (include/helrm.h) -- argument
marshalling only: every step of the lookup runs in the library's sm_100a
kernels.  Names follow the C ABI without the `helrm_` prefix.

There is no fallback: if the shared library is missing, importing this module
raises (build it with `python -m paper_2506_18150_b200.build` or
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HELRM_LIB") or os.path.join(_HERE, "lib", "libhelrm.so")   # override: A/B experiments

HELRM_OK = 0
ERRORS = {2: "CONFIG", 3: "LEVEL", 4: "CAPACITY", 5: "RANGE", 6: "LAYOUT", 7: "CUDA", 8: "NCCL", 9: "ALLOC", 10: "ARG"}
MODE_DOUBLE, MODE_SINGLE = 0, 1

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libhelrm.so not built ({LIB_PATH}); run __graft_entry__.build()")
_L = ctypes.CDLL(LIB_PATH)


class HelrmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"HELRM_ERR_{ERRORS.get(code, code)}: {msg}")
        self.code = code


class ParamsDesc(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n_q_groups", ctypes.c_uint32), ("q_bits", ctypes.c_uint32 * 8),
                ("q_count", ctypes.c_uint32 * 8), ("n_p_groups", ctypes.c_uint32), ("p_bits", ctypes.c_uint32 * 4),
                ("p_count", ctypes.c_uint32 * 4), ("log_scale", ctypes.c_uint32)]


class ParamsInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("N", "n_slots", "L", "K", "dnum_top", "log_scale")]


class TableDesc(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("d", ctypes.c_int64), ("p", ctypes.c_int64),
                ("w", ctypes.POINTER(ctypes.c_double)), ("in_off", ctypes.c_int64), ("out_off", ctypes.c_int64),
                ("l", ctypes.c_int64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("K", "M", "mbar", "n_in_cts", "n_out_cts", "n_diag", "n_unique", "n1",
                                              "n2_max", "n_rotations")] + \
               [("level", ctypes.c_uint32), ("mode", ctypes.c_uint32), ("diag_bytes", ctypes.c_uint64)]


_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_sz = ctypes.c_size_t
_i64 = ctypes.c_int64
_pp = ctypes.POINTER(ctypes.c_void_p)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "helrm_params_create": [ctypes.POINTER(ParamsDesc), _pp],
    "helrm_params_info": [_vp, ctypes.POINTER(ParamsInfo)],
    "helrm_params_moduli": [_vp, _u64p, _u64p, _u64p],
    "helrm_ctx_create": [_vp, ctypes.c_int, ctypes.c_size_t, _pp],
    "helrm_ctx_sync": [_vp],
    "helrm_sk_gen": [_vp, _u64, _pp],
    "helrm_pk_gen": [_vp, _vp, _u64, _pp],
    "helrm_rotkeys_gen": [_vp, _vp, _u64p, _sz, _u64, _pp],
    "helrm_sk_export": [_vp, _vp, _i64p, _sz],
    "helrm_pk_export": [_vp, _vp, _u64p, _sz],
    "helrm_rotkeys_export": [_vp, _vp, _u64, _u64p, _sz],
    "helrm_tables_create": [_vp, ctypes.POINTER(TableDesc), _sz, _u32, _pp],
    "helrm_tables_info": [_vp, _i64p, _i64p],
    "helrm_encode_query": [_vp, _i64p, _dp, _dp, _sz],
    "helrm_encrypt": [_vp, _vp, _dp, _sz, _u32, _u64, _pp],
    "helrm_ct_import": [_vp, _u64p, _u32, ctypes.c_double, _pp],
    "helrm_ct_export": [_vp, _vp, _u64p, _sz],
    "helrm_ct_info": [_vp, ctypes.POINTER(_u32), _dp],
    "helrm_ct_device_ptr": [_vp, ctypes.POINTER(_u64p)],
    "helrm_ct_alloc": [_vp, _u32, ctypes.c_double, _pp],
    "helrm_ct_random": [_vp, _u64, _u32, _u32, _pp],
    "helrm_decrypt_decode": [_vp, _vp, _vp, _dp, _sz],
    "helrm_plan_create": [_vp, _vp, _u32, _u32, _u32, _pp],
    "helrm_plan_info": [_vp, ctypes.POINTER(PlanInfo)],
    "helrm_plan_rotations": [_vp, _i64p, _sz, ctypes.POINTER(_sz)],
    "helrm_lookup": [_vp, _vp, _vp, _pp, _sz, _pp],
    "helrm_lookup_host": [_vp, _vp, _vp, _pp, ctypes.c_double, _sz, _pp],
    "helrm_ntt_fwd": [_vp, _vp, _u32, _u32, _sz],
    "helrm_ntt_inv": [_vp, _vp, _u32, _u32, _sz],
    "helrm_modup": [_vp, _vp, _u32, _u32, _vp],
    "helrm_moddown": [_vp, _vp, _u32, _vp],
    "helrm_rescale": [_vp, _vp, _pp],
    "helrm_rotate": [_vp, _vp, _vp, _i64, _pp],
    "helrm_rotate_hoisted": [_vp, _vp, _vp, _i64p, _sz, _pp, _sz],
    "helrm_rotate_hoisted_batch": [_vp, _vp, _pp, _sz, _i64p, _sz, _vp, _sz],
    "helrm_dist_range": [_i64, ctypes.c_int, ctypes.c_int, _i64p, _i64p],
    "helrm_comm_unique_id": [ctypes.POINTER(ctypes.c_uint8)],
    "helrm_comm_init": [_vp, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int, ctypes.c_int],
    "helrm_lookup_dist": [_vp, _vp, _vp, _pp, _sz, _pp],
    "helrm_lookup_dist_virtual": [_vp, _vp, _vp, _pp, _sz, ctypes.c_int, _pp],
    "helrm_modred": [_vp, _vp, _u32, _sz],
    "helrm_lookup_limbsplit_virtual": [_vp, _vp, _vp, _pp, _sz, ctypes.c_int, _pp],
    "helrm_lookup_limbsplit": [_vp, _vp, _vp, _pp, _sz, _pp],
    "helrm_limbsplit_rank_work": [_vp, _vp, _vp, _pp, ctypes.c_int, ctypes.c_int, _pp],
    "helrm_plan_galois": [_vp, _u64p, _sz, ctypes.POINTER(_sz)],
    "helrm_rotkeys_galois": [_vp, _u64p, _sz, ctypes.POINTER(_sz)],
    "helrm_sk_import": [_vp, _i64p, _sz, _pp],
    "helrm_pk_import": [_vp, _u64p, _sz, _pp],
    "helrm_rotkeys_import": [_vp, _u64p, _sz, _pp, _sz, _pp],
    "helrm_rotkeys_upload": [_vp, _vp, _u64, _u64p, _sz],
}
for _name, _args in _SIGS.items():
    _f = getattr(_L, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
for _name in ("helrm_params_destroy", "helrm_ctx_destroy", "helrm_sk_destroy", "helrm_pk_destroy",
              "helrm_rotkeys_destroy", "helrm_tables_destroy", "helrm_ct_destroy", "helrm_plan_destroy"):
    getattr(_L, _name).argtypes = [_vp]
    getattr(_L, _name).restype = None
_L.helrm_last_error.restype = ctypes.c_char_p
_L.helrm_version.restype = ctypes.c_char_p
_L.helrm_ctx_launches.argtypes = [_vp]
_L.helrm_ctx_launches.restype = _u64
_L.helrm_ctx_profile.argtypes = [_vp, ctypes.c_int]
_L.helrm_ctx_profile.restype = ctypes.c_int
_L.helrm_ctx_profile_json.argtypes = [_vp]
_L.helrm_ctx_profile_json.restype = ctypes.c_char_p
_L.helrm_rotkeys_bytes.argtypes = [_vp]
_L.helrm_rotkeys_bytes.restype = _sz

EXPORTED = sorted(list(_SIGS) + ["helrm_params_destroy", "helrm_ctx_destroy", "helrm_sk_destroy", "helrm_pk_destroy",
                                 "helrm_rotkeys_destroy", "helrm_tables_destroy", "helrm_ct_destroy",
                                 "helrm_plan_destroy", "helrm_last_error", "helrm_version", "helrm_ctx_launches",
                                 "helrm_rotkeys_bytes", "helrm_ctx_profile", "helrm_ctx_profile_json", "helrm_dist_range",
                                 "helrm_comm_unique_id", "helrm_comm_init", "helrm_lookup_dist",
                                 "helrm_lookup_dist_virtual", "helrm_modred", "helrm_plan_galois",
                                 "helrm_lookup_limbsplit_virtual", "helrm_lookup_limbsplit",
                                 "helrm_limbsplit_rank_work", "helrm_rotate_hoisted_batch",
                                 "helrm_rotkeys_galois", "helrm_sk_import", "helrm_pk_import",
                                 "helrm_rotkeys_import", "helrm_rotkeys_upload"])


def _check(code: int):
    if code != HELRM_OK:
        raise HelrmError(code, _L.helrm_last_error().decode())


def version() -> str:
    return _L.helrm_version().decode()


def _u64ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _devptr(t) -> int:
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


class _Handle:
    _destroy = None

    def __init__(self, h: ctypes.c_void_p, owner=None):
        self.h = h
        self._owner = owner        # keeps the context alive while this handle lives
        if owner is not None and hasattr(owner, "_children"):
            owner._children.add(self)   # the C ABI needs every handle destroyed before its context

    def close(self):
        if self.h:
            getattr(_L, self._destroy)(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- params
class Params(_Handle):
    _destroy = "helrm_params_destroy"

    def info(self) -> ParamsInfo:
        i = ParamsInfo()
        _check(_L.helrm_params_info(self.h, ctypes.byref(i)))
        return i

    def moduli(self):
        i = self.info()
        q = np.zeros(i.L + 1, np.uint64)
        p = np.zeros(i.K, np.uint64)
        psi = np.zeros(i.L + 1 + i.K, np.uint64)
        _check(_L.helrm_params_moduli(self.h, _u64ptr(q), _u64ptr(p), _u64ptr(psi)))
        return [int(x) for x in q], [int(x) for x in p], [int(x) for x in psi]


def params_create(log_n: int, q_groups, p_groups, log_scale: int) -> Params:
    d = ParamsDesc()
    d.log_n = log_n
    d.n_q_groups = len(q_groups)
    for i, (b, c) in enumerate(q_groups):
        d.q_bits[i], d.q_count[i] = b, c
    d.n_p_groups = len(p_groups)
    for i, (b, c) in enumerate(p_groups):
        d.p_bits[i], d.p_count[i] = b, c
    d.log_scale = log_scale
    h = ctypes.c_void_p()
    _check(_L.helrm_params_create(ctypes.byref(d), ctypes.byref(h)))
    return Params(h)


def params_from_config(cfg) -> Params:
    return params_create(cfg.log_n, cfg.q_groups, cfg.p_groups, cfg.log_scale)


# ---------------------------------------------------------------- tables
class Tables(_Handle):
    _destroy = "helrm_tables_destroy"

    def info(self):
        K, M = ctypes.c_int64(), ctypes.c_int64()
        _check(_L.helrm_tables_info(self.h, ctypes.byref(K), ctypes.byref(M)))
        return K.value, M.value


def tables_create(params: Params, tables: Sequence, n_dense: int) -> Tables:
    """tables: objects with k, d, p, weights (float64 rows x d), in_off, out_off, l."""
    keep = []
    arr = (TableDesc * len(tables))()
    seen = {}
    for i, t in enumerate(tables):
        w = seen.get(id(t.weights))
        if w is None:
            w = np.ascontiguousarray(t.weights, dtype=np.float64)
            seen[id(t.weights)] = w
            keep.append(w)
        arr[i].k, arr[i].d, arr[i].p = t.k, t.d, t.p
        arr[i].w = _dptr(w)
        arr[i].in_off, arr[i].out_off = getattr(t, "in_off", -1), getattr(t, "out_off", -1)
        arr[i].l = getattr(t, "l", 0)
    h = ctypes.c_void_p()
    _check(_L.helrm_tables_create(params.h, arr, len(tables), n_dense, ctypes.byref(h)))
    return Tables(h)


def encode_query(tables: Tables, idx, dense, n_slots: int) -> np.ndarray:
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    dense = np.ascontiguousarray(dense if dense is not None else np.zeros(0), dtype=np.float64)
    out = np.zeros(n_slots)
    _check(_L.helrm_encode_query(tables.h, idx.ctypes.data_as(_i64p), _dptr(dense) if dense.size else None,
                                 _dptr(out), n_slots))
    return out


# ---------------------------------------------------------------- context and keys
class Context(_Handle):
    _destroy = "helrm_ctx_destroy"

    def __init__(self, params: Params, device: int = 0, stream: int = 0):
        import weakref
        h = ctypes.c_void_p()
        _check(_L.helrm_ctx_create(params.h, device, stream, ctypes.byref(h)))
        self._children = weakref.WeakSet()
        super().__init__(h)
        self.params = params
        self.info = params.info()

    def close(self):
        """Destroy the context after every handle created on it (ciphertexts,
        keys, plans) that is still alive: helrm_ctx_destroy frees the device
        memory pool those handles live in."""
        if self.h:
            for ch in list(self._children):
                ch.close()
        super().close()

    def sync(self):
        _check(_L.helrm_ctx_sync(self.h))

    def launches(self) -> int:
        return int(_L.helrm_ctx_launches(self.h))

    def profile(self, on: bool):
        _check(_L.helrm_ctx_profile(self.h, 1 if on else 0))

    def profile_stats(self) -> dict:
        import json
        return json.loads(_L.helrm_ctx_profile_json(self.h).decode())


class SecretKey(_Handle):
    _destroy = "helrm_sk_destroy"


class PublicKey(_Handle):
    _destroy = "helrm_pk_destroy"


class RotKeys(_Handle):
    _destroy = "helrm_rotkeys_destroy"

    def nbytes(self) -> int:
        return int(_L.helrm_rotkeys_bytes(self.h))

    def galois(self) -> List[int]:
        n = ctypes.c_size_t()
        _check(_L.helrm_rotkeys_galois(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.uint64)
        _check(_L.helrm_rotkeys_galois(self.h, _u64ptr(out) if out.size else None, out.size, ctypes.byref(n)))
        return [int(x) for x in out]


def ctx_create(params: Params, device: int = 0, stream: int = 0) -> Context:
    return Context(params, device, stream)


def sk_gen(ctx: Context, seed: int) -> SecretKey:
    h = ctypes.c_void_p()
    _check(_L.helrm_sk_gen(ctx.h, seed, ctypes.byref(h)))
    return SecretKey(h, ctx)


def pk_gen(ctx: Context, sk: SecretKey, seed: int) -> PublicKey:
    h = ctypes.c_void_p()
    _check(_L.helrm_pk_gen(ctx.h, sk.h, seed, ctypes.byref(h)))
    return PublicKey(h, ctx)


def rotkeys_gen(ctx: Context, sk: SecretKey, galois: Sequence[int], seed: int) -> RotKeys:
    g = np.ascontiguousarray(np.array(list(galois), dtype=np.uint64))
    h = ctypes.c_void_p()
    _check(_L.helrm_rotkeys_gen(ctx.h, sk.h, _u64ptr(g) if g.size else None, g.size, seed, ctypes.byref(h)))
    return RotKeys(h, ctx)


def sk_import(ctx: Context, coeff: np.ndarray) -> SecretKey:
    a = np.ascontiguousarray(coeff, dtype=np.int64)
    h = ctypes.c_void_p()
    _check(_L.helrm_sk_import(ctx.h, a.ctypes.data_as(_i64p), a.size, ctypes.byref(h)))
    return SecretKey(h, ctx)


def pk_import(ctx: Context, coeff: np.ndarray) -> PublicKey:
    a = np.ascontiguousarray(coeff, dtype=np.uint64)
    h = ctypes.c_void_p()
    _check(_L.helrm_pk_import(ctx.h, _u64ptr(a), a.size, ctypes.byref(h)))
    return PublicKey(h, ctx)


def rotkeys_import(ctx: Context, keys: dict) -> RotKeys:
    """keys: {galois element: uint64 [dnum][2][L+1+K][N] coefficient form}."""
    gs = np.array(list(keys), dtype=np.uint64)
    arrs = [np.ascontiguousarray(keys[int(g)], dtype=np.uint64) for g in gs]
    wpk = min((a.size for a in arrs), default=0)
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    h = ctypes.c_void_p()
    _check(_L.helrm_rotkeys_import(ctx.h, _u64ptr(gs) if gs.size else None, gs.size, ptrs, wpk, ctypes.byref(h)))
    return RotKeys(h, ctx)


def rotkeys_upload(ctx: Context, rk: RotKeys, g: int, coeff: np.ndarray) -> None:
    a = np.ascontiguousarray(coeff, dtype=np.uint64)
    _check(_L.helrm_rotkeys_upload(ctx.h, rk.h, g, _u64ptr(a), a.size))


def sk_export(ctx: Context, sk: SecretKey) -> np.ndarray:
    out = np.zeros(ctx.info.N, np.int64)
    _check(_L.helrm_sk_export(ctx.h, sk.h, out.ctypes.data_as(_i64p), out.size))
    return out


def pk_export(ctx: Context, pk: PublicKey) -> np.ndarray:
    i = ctx.info
    out = np.zeros((2, i.L + 1, i.N), np.uint64)
    _check(_L.helrm_pk_export(ctx.h, pk.h, _u64ptr(out), out.size))
    return out


def rotkeys_export(ctx: Context, rk: RotKeys, g: int) -> np.ndarray:
    i = ctx.info
    out = np.zeros((i.dnum_top, 2, i.L + 1 + i.K, i.N), np.uint64)
    _check(_L.helrm_rotkeys_export(ctx.h, rk.h, g, _u64ptr(out), out.size))
    return out


# ---------------------------------------------------------------- ciphertexts
class Ciphertext(_Handle):
    _destroy = "helrm_ct_destroy"

    def info(self):
        lv, sc = _u32(), ctypes.c_double()
        _check(_L.helrm_ct_info(self.h, ctypes.byref(lv), ctypes.byref(sc)))
        return lv.value, sc.value

    @property
    def level(self) -> int:
        return self.info()[0]

    def device_ptr(self) -> int:
        p = _u64p()
        _check(_L.helrm_ct_device_ptr(self.h, ctypes.byref(p)))
        return ctypes.cast(p, ctypes.c_void_p).value


def encrypt(ctx: Context, pk: PublicKey, slots: np.ndarray, level: int, seed: int) -> Ciphertext:
    z = np.ascontiguousarray(slots, dtype=np.float64)
    h = ctypes.c_void_p()
    _check(_L.helrm_encrypt(ctx.h, pk.h, _dptr(z), z.size, level, seed, ctypes.byref(h)))
    return Ciphertext(h, ctx)


def ct_import(ctx: Context, coeff: np.ndarray, level: int, scale: float) -> Ciphertext:
    a = np.ascontiguousarray(coeff, dtype=np.uint64)
    assert a.size == 2 * (level + 1) * ctx.info.N
    h = ctypes.c_void_p()
    _check(_L.helrm_ct_import(ctx.h, _u64ptr(a), level, float(scale), ctypes.byref(h)))
    return Ciphertext(h, ctx)


def ct_export(ctx: Context, ct: Ciphertext) -> np.ndarray:
    lv = ct.level
    out = np.zeros((2, lv + 1, ctx.info.N), np.uint64)
    _check(_L.helrm_ct_export(ctx.h, ct.h, _u64ptr(out), out.size))
    return out


def ct_alloc(ctx: Context, level: int, scale: float = 1.0) -> Ciphertext:
    h = ctypes.c_void_p()
    _check(_L.helrm_ct_alloc(ctx.h, level, scale, ctypes.byref(h)))
    return Ciphertext(h, ctx)


def ct_random(ctx: Context, seed: int, index: int, level: int) -> Ciphertext:
    h = ctypes.c_void_p()
    _check(_L.helrm_ct_random(ctx.h, seed, index, level, ctypes.byref(h)))
    return Ciphertext(h, ctx)


def decrypt_decode(ctx: Context, sk: SecretKey, ct: Ciphertext, n_slots: Optional[int] = None) -> np.ndarray:
    n = ctx.info.n_slots if n_slots is None else n_slots
    out = np.zeros(n)
    _check(_L.helrm_decrypt_decode(ctx.h, sk.h, ct.h, _dptr(out), n))
    return out


# ---------------------------------------------------------------- plan and lookup
class Plan(_Handle):
    _destroy = "helrm_plan_destroy"

    def info(self) -> PlanInfo:
        i = PlanInfo()
        _check(_L.helrm_plan_info(self.h, ctypes.byref(i)))
        return i

    def rotations(self) -> List[int]:
        n = ctypes.c_size_t()
        _check(_L.helrm_plan_rotations(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.int64)
        _check(_L.helrm_plan_rotations(self.h, out.ctypes.data_as(_i64p), out.size, ctypes.byref(n)))
        return [int(x) for x in out]

    def galois(self, N: Optional[int] = None) -> List[int]:
        """helrm_plan_galois: the D19 Galois list, computed by the library
        (N is accepted for backwards compatibility and ignored)."""
        n = ctypes.c_size_t()
        _check(_L.helrm_plan_galois(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.uint64)
        _check(_L.helrm_plan_galois(self.h, _u64ptr(out) if out.size else None, out.size, ctypes.byref(n)))
        return [int(x) for x in out]


def plan_create(ctx: Context, tables: Tables, level: int, n1: int = 0, mode: int = MODE_DOUBLE) -> Plan:
    h = ctypes.c_void_p()
    _check(_L.helrm_plan_create(ctx.h, tables.h, level, n1, mode, ctypes.byref(h)))
    return Plan(h, ctx)


def lookup(ctx: Context, plan: Plan, rk: RotKeys, cts: Sequence[Ciphertext], batch: int = 1) -> List[Ciphertext]:
    info = plan.info()
    assert len(cts) == batch * info.n_in_cts
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    outs = (ctypes.c_void_p * (batch * info.n_out_cts))()
    _check(_L.helrm_lookup(ctx.h, plan.h, rk.h, ins, batch, outs))
    return [Ciphertext(ctypes.c_void_p(o), ctx) for o in outs]


def lookup_host(ctx: Context, plan: Plan, rk: RotKeys, inputs: Sequence, scale: float, batch: int,
                outputs: Sequence) -> None:
    """helrm_lookup_host: `inputs` = batch x C host arrays (coefficient form
    [2][level+1][N] uint64, pinned for asynchronous copies), `outputs` =
    batch x O host arrays [2][level][N] filled in place."""
    info = plan.info()
    assert len(inputs) == batch * info.n_in_cts and len(outputs) == batch * info.n_out_cts
    for a in list(inputs) + list(outputs):
        assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    ins = (ctypes.c_void_p * len(inputs))(*[a.ctypes.data for a in inputs])
    outs = (ctypes.c_void_p * len(outputs))(*[a.ctypes.data for a in outputs])
    _check(_L.helrm_lookup_host(ctx.h, plan.h, rk.h, ins, float(scale), batch, outs))


# ---------------------------------------------------------------- primitives
def ntt_fwd(ctx: Context, dev, first_prime: int, n_limbs: int, n_polys: int = 1):
    _check(_L.helrm_ntt_fwd(ctx.h, _devptr(dev), first_prime, n_limbs, n_polys))


def ntt_inv(ctx: Context, dev, first_prime: int, n_limbs: int, n_polys: int = 1):
    _check(_L.helrm_ntt_inv(ctx.h, _devptr(dev), first_prime, n_limbs, n_polys))


def modup(ctx: Context, dev_in, level: int, digit: int, dev_out):
    _check(_L.helrm_modup(ctx.h, _devptr(dev_in), level, digit, _devptr(dev_out)))


def moddown(ctx: Context, dev_in, level: int, dev_out):
    _check(_L.helrm_moddown(ctx.h, _devptr(dev_in), level, _devptr(dev_out)))


def rescale(ctx: Context, ct: Ciphertext) -> Ciphertext:
    h = ctypes.c_void_p()
    _check(_L.helrm_rescale(ctx.h, ct.h, ctypes.byref(h)))
    return Ciphertext(h, ctx)


def rotate(ctx: Context, rk: RotKeys, ct: Ciphertext, k: int) -> Ciphertext:
    h = ctypes.c_void_p()
    _check(_L.helrm_rotate(ctx.h, rk.h, ct.h, k, ctypes.byref(h)))
    return Ciphertext(h, ctx)


def rotate_hoisted(ctx: Context, rk: RotKeys, ct: Ciphertext, amounts: Sequence[int], ring: Sequence[Ciphertext]):
    a = np.ascontiguousarray(np.array(list(amounts), dtype=np.int64))
    r = (ctypes.c_void_p * len(ring))(*[c.h for c in ring])
    _check(_L.helrm_rotate_hoisted(ctx.h, rk.h, ct.h, a.ctypes.data_as(_i64p), a.size, r, len(ring)))


def rotate_hoisted_batch(ctx: Context, rk: RotKeys, cts: Sequence[Ciphertext], amounts: Sequence[int], dev_out,
                         ring: int):
    """helrm_rotate_hoisted_batch: Rotate(cts[j], amounts[i]) -> dev_out slot (i n + j) % ring,
    [ring][2][level+1][N] uint64 (NTT slot order)."""
    a = np.ascontiguousarray(np.array(list(amounts), dtype=np.int64))
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    _check(_L.helrm_rotate_hoisted_batch(ctx.h, rk.h, ins, len(cts), a.ctypes.data_as(_i64p), a.size, _devptr(dev_out),
                                         ring))


# ---------------------------------------------------------------- multi-GPU
def dist_range(n_items: int, world: int, rank: int):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(_L.helrm_dist_range(n_items, world, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_L.helrm_comm_unique_id(buf))
    return bytes(buf)


def comm_init(ctx: Context, uid: bytes, rank: int, world: int):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(_L.helrm_comm_init(ctx.h, buf, rank, world))


def lookup_dist_virtual(ctx: Context, plan: Plan, rk: RotKeys, cts: Sequence[Ciphertext], parts: int,
                        batch: int = 1) -> List[Ciphertext]:
    info = plan.info()
    assert len(cts) == batch * info.n_in_cts
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    outs = (ctypes.c_void_p * (batch * info.n_out_cts))()
    _check(_L.helrm_lookup_dist_virtual(ctx.h, plan.h, rk.h, ins, batch, parts, outs))
    return [Ciphertext(ctypes.c_void_p(o), ctx) for o in outs]


def lookup_limbsplit_virtual(ctx: Context, plan: Plan, rk: RotKeys, cts: Sequence[Ciphertext], parts: int,
                             batch: int = 1) -> List[Ciphertext]:
    info = plan.info()
    assert len(cts) == batch * info.n_in_cts
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    outs = (ctypes.c_void_p * (batch * info.n_out_cts))()
    _check(_L.helrm_lookup_limbsplit_virtual(ctx.h, plan.h, rk.h, ins, batch, parts, outs))
    return [Ciphertext(ctypes.c_void_p(o), ctx) for o in outs]


def lookup_limbsplit(ctx: Context, plan: Plan, rk: RotKeys, cts: Sequence[Ciphertext], batch: int = 1) -> List[Ciphertext]:
    info = plan.info()
    assert len(cts) == batch * info.n_in_cts
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    outs = (ctypes.c_void_p * (batch * info.n_out_cts))()
    _check(_L.helrm_lookup_limbsplit(ctx.h, plan.h, rk.h, ins, batch, outs))
    return [Ciphertext(ctypes.c_void_p(o), ctx) for o in outs]


def limbsplit_rank_work(ctx: Context, plan: Plan, rk: RotKeys, cts: Sequence[Ciphertext], parts: int,
                        rank: int) -> List[Ciphertext]:
    """Timing harness: rank `rank`'s kernels of the limb partition (outputs are not a lookup)."""
    info = plan.info()
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    outs = (ctypes.c_void_p * info.n_out_cts)()
    _check(_L.helrm_limbsplit_rank_work(ctx.h, plan.h, rk.h, ins, parts, rank, outs))
    return [Ciphertext(ctypes.c_void_p(o), ctx) for o in outs]


def modred(ctx: Context, dev, level: int, n_polys: int = 1):
    _check(_L.helrm_modred(ctx.h, _devptr(dev), level, n_polys))


def lookup_dist(ctx: Context, plan: Plan, rk: RotKeys, cts: Sequence[Ciphertext], batch: int = 1) -> List[Ciphertext]:
    info = plan.info()
    assert len(cts) == batch * info.n_in_cts
    ins = (ctypes.c_void_p * len(cts))(*[c.h for c in cts])
    outs = (ctypes.c_void_p * (batch * info.n_out_cts))()
    _check(_L.helrm_lookup_dist(ctx.h, plan.h, rk.h, ins, batch, outs))
    return [Ciphertext(ctypes.c_void_p(o), ctx) for o in outs]
