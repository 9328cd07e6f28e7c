"""ctypes front-ends for the two CPU checkers. TEST INFRASTRUCTURE ONLY.

* ``Port`` wraps ``oracle/liboomb_oracle.so`` — the plain-C restatement of the
  reference hot path (``oracle/oomb_oracle.c``), built from this repository.
* ``Ref`` wraps ``oracle/_ref/libchunktrain_ref.so`` — the UNMODIFIED reference
  headers compiled in place from /root/reference (``oracle/Makefile.ref``), when
  that build exists.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module; the product package never does.
Both classes expose the same Python surface so a test can run an identical
script through either and compare bit patterns.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboomb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchunktrain_ref.so")

ERRORS = {1: "ConfigError", 2: "ShapeError", 3: "StateError", 4: "ResidencyError", 5: "IoError", 9: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")


def _p(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def build_port(force: bool = False) -> str:
    """Compile the C restatement (gcc, -ffp-contract=off, no -march=native)."""
    src = os.path.join(HERE, "oomb_oracle.c")
    if force or not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
        cmd = f"gcc -std=c11 -O2 -g -fPIC -ffp-contract=off -shared -o {PORT_SO} {src} -lm"
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
    return PORT_SO


def build_ref(force: bool = False) -> str | None:
    """Compile oracle/_ref from /root/reference when the reference is present."""
    if not os.path.isdir("/root/reference/proj"):
        return REF_SO if os.path.exists(REF_SO) else None
    mk = os.path.join(HERE, "Makefile.ref")
    if force:
        os.system(f"make -s -f {mk} clean")
    if os.system(f"make -s -f {mk}") != 0:
        raise RuntimeError("reference shim build failed")
    return REF_SO


@dataclass
class Cfg:
    n_layers: int = 1
    n_q_heads: int = 4
    n_kv_heads: int = 2
    head_dim: int = 8
    chunk_size: int = 16
    page_size: int = 8
    retrieval_budget: int = 16
    local_window: int = 4
    score_scale: int = 0

    @property
    def gqa_group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def pages_per_chunk(self) -> int:
        return self.chunk_size // self.page_size

    @property
    def budget_pages(self) -> int:
        return self.retrieval_budget // self.page_size


class _RefCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_layers", "n_q_heads", "n_kv_heads", "head_dim", "chunk_size",
                                         "page_size", "retrieval_budget", "local_window", "score_scale")]


class RefEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("page", C.c_int32), ("chunk", C.c_int32),
                ("phase", C.c_int32), ("pad", C.c_int32), ("bytes", C.c_uint64), ("t", C.c_double)]


def csr(lists) -> tuple[np.ndarray, np.ndarray]:
    off = np.zeros(len(lists) + 1, dtype=np.int32)
    for i, l in enumerate(lists):
        off[i + 1] = off[i] + len(l)
    ids = np.concatenate([np.asarray(l, dtype=np.int32) for l in lists]) if off[-1] else np.zeros(0, np.int32)
    return off, _i32(ids)


class _Base:
    """Common numpy-facing surface; subclasses bind the C symbols."""

    dtype: np.dtype
    cfg: Cfg

    def _chk(self, rc: int):
        if rc:
            raise OracleError(rc, self._err().decode(errors="replace"))

    def _a(self, x) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(x, dtype=self.dtype))

    # ---- shapes -------------------------------------------------------------
    @property
    def row_elems(self) -> int:
        return self.cfg.n_kv_heads * self.cfg.head_dim


class Port(_Base):
    """The C restatement (oracle/oomb_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(build_port())
            L.oc_last_error.restype = C.c_char_p
            L.oc_cache_filled.restype = C.c_int64
            cls._lib = L
        return cls._lib

    def __init__(self, cfg: Cfg, real_bytes: int = 4):
        self.L = self.lib()
        self.cfg = cfg
        self.real_bytes = real_bytes
        self.dtype = np.dtype(np.float32 if real_bytes == 4 else np.float64)
        self.suf = "f32" if real_bytes == 4 else "f64"
        self._err = self.L.oc_last_error
        self._chk(self.L.oc_validate(cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.chunk_size,
                                     cfg.page_size, cfg.retrieval_budget, cfg.local_window))
        h = C.c_void_p()
        self._chk(self.L.oc_cache_new(real_bytes, cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.page_size,
                                      C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.oc_cache_free(self.h)
            self.h = None

    def fn(self, name):
        return getattr(self.L, f"oc_{name}_{self.suf}")

    # ---- page manager -------------------------------------------------------
    def append(self, layer, k, v):
        k, v = self._a(k), self._a(v)
        b, e = C.c_int64(), C.c_int64()
        self._chk(self.fn("append")(self.h, layer, _p(k), _p(v), C.c_int64(k.shape[0]), C.byref(b), C.byref(e)))
        return b.value, e.value

    def n_pages(self, layer):
        return self.L.oc_cache_n_pages(self.h, layer)

    def filled(self, layer):
        return self.L.oc_cache_filled(self.h, layer)

    def page_table(self, layer) -> np.ndarray:
        n = max(self.n_pages(layer), 0)
        out = np.zeros((n, 4), np.int32)
        self._chk(self.L.oc_cache_page_table(self.h, layer, _p(out)))
        return out

    def kavg_raw(self, layer):
        n = self.n_pages(layer)
        s = np.zeros((n, self.cfg.n_kv_heads, self.cfg.head_dim), self.dtype)
        cnt = np.zeros(n, np.int32)
        self._chk(self.L.oc_cache_kavg_raw(self.h, layer, _p(s), _p(cnt)))
        return s, cnt

    def mean_keys(self, layer, n=-1):
        cap = max(self.n_pages(layer), 0)
        out = np.zeros((cap, self.cfg.n_kv_heads, self.cfg.head_dim), self.dtype)
        no = C.c_int()
        self._chk(self.fn("mean_keys")(self.h, layer, n, _p(out), C.byref(no)))
        return out[: no.value]

    def gather(self, layer, ids, grads=False):
        ids = _i32(ids)
        rows = len(ids) * self.cfg.page_size
        k = np.zeros((rows, self.cfg.n_kv_heads, self.cfg.head_dim), self.dtype)
        v = np.zeros_like(k)
        valid = np.zeros(rows, np.uint8)
        self._chk(self.fn("gather")(self.h, layer, _p(ids), len(ids), int(grads), _p(k), _p(v), _p(valid)))
        return k, v, valid

    def scatter(self, layer, ids, dk, dv):
        ids = _i32(ids)
        dk, dv = self._a(dk), self._a(dv)
        if dk.shape[0] != len(ids) * self.cfg.page_size:
            raise OracleError(2, "scatter_add_grads: gradient shape does not match gather layout")
        self._chk(self.fn("scatter")(self.h, layer, _p(ids), len(ids), _p(dk), _p(dv)))

    def reset(self):
        self.L.oc_cache_reset(self.h)

    def zero_grad(self):
        self.L.oc_cache_zero_grad(self.h)

    def set_tier(self, layer, page, tier):
        self._chk(self.L.oc_cache_set_tier(self.h, layer, page, tier))

    def set_residency_enforced(self, on):
        self.L.oc_cache_set_residency_enforced(self.h, int(on))

    def memory_report(self) -> dict:
        out = np.zeros(8, np.uint64)
        self.L.oc_cache_memory_report(self.h, _p(out))
        return _report(out)

    # ---- attention ----------------------------------------------------------
    def score_pages(self, q, k_avg, score_scale=None):
        q, k_avg = self._a(q), self._a(k_avg)
        cfg = self.cfg
        m = (q.shape[0] + cfg.page_size - 1) // cfg.page_size
        out = np.zeros((m, k_avg.shape[0]), self.dtype)
        sc = cfg.score_scale if score_scale is None else int(score_scale)
        self._chk(self.fn("score_pages")(_p(q), C.c_int64(q.shape[0]), q.shape[1], q.shape[2], _p(k_avg),
                                         C.c_int64(k_avg.shape[0]), k_avg.shape[1], cfg.page_size,
                                         q.shape[1] // k_avg.shape[1], sc, _p(out)))
        return out

    def attn_forward(self, layer, q, selected, k_cur, v_cur):
        q, k_cur, v_cur = self._a(q), self._a(k_cur), self._a(v_cur)
        off, ids = csr(selected)
        out = np.zeros_like(q)
        lse = np.zeros(q.shape[:2], self.dtype)
        self._chk(self.fn("attn_forward")(self.h, layer, q.shape[1], _p(q), C.c_int64(q.shape[0]), _p(off),
                                          _p(ids), C.c_int64(len(selected)), _p(k_cur), _p(v_cur), _p(out),
                                          _p(lse)))
        return out, lse

    def attn_backward(self, layer, dout, q, selected, k_cur, v_cur, out, lse):
        dout, q, k_cur, v_cur, out, lse = map(self._a, (dout, q, k_cur, v_cur, out, lse))
        off, ids = csr(selected)
        dq = np.zeros_like(q)
        dk = np.zeros_like(k_cur)
        dv = np.zeros_like(v_cur)
        self._chk(self.fn("attn_backward")(self.h, layer, q.shape[1], _p(dout), _p(q), C.c_int64(q.shape[0]),
                                           _p(off), _p(ids), C.c_int64(len(selected)), _p(k_cur), _p(v_cur),
                                           _p(out), _p(lse), _p(dq), _p(dk), _p(dv)))
        return dq, dk, dv

    def naive_attention(self, q, k, v, past_len, dout, gqa_group):
        q, k, v, dout = map(self._a, (q, k, v, dout))
        out, dq = np.zeros_like(q), np.zeros_like(q)
        dk, dv = np.zeros_like(k), np.zeros_like(v)
        self._chk(self.fn("naive_attention")(_p(q), C.c_int64(q.shape[0]), q.shape[1], q.shape[2], _p(k), _p(v),
                                             C.c_int64(k.shape[0]), k.shape[1], C.c_int64(past_len), _p(dout),
                                             gqa_group, _p(out), _p(dq), _p(dk), _p(dv)))
        return out, dq, dk, dv

    # ---- selection (type-free) ----------------------------------------------
    @classmethod
    def select_topk(cls, row, budget) -> np.ndarray:
        L = cls.lib()
        row = np.ascontiguousarray(np.asarray(row, dtype=np.float64))
        out = np.zeros(max(len(row), 1), np.int32)
        cnt = C.c_int()
        rc = L.oc_select_topk(_p(row), len(row), int(budget), _p(out), C.byref(cnt))
        if rc:
            raise OracleError(rc, L.oc_last_error().decode())
        return out[: cnt.value]

    @classmethod
    def select_recent(cls, n_pages, window) -> np.ndarray:
        L = cls.lib()
        out = np.zeros(max(n_pages, 1), np.int32)
        cnt = C.c_int()
        rc = L.oc_select_recent(n_pages, window, _p(out), C.byref(cnt))
        if rc:
            raise OracleError(rc, L.oc_last_error().decode())
        return out[: cnt.value]


def _report(out: np.ndarray) -> dict:
    keys = ("device_bytes", "host_bytes", "grad_bytes", "pages", "reallocs", "copied_bytes", "arena_blocks",
            "free_list")
    return {k: int(v) for k, v in zip(keys, out)}


class Ref(_Base):
    """The reference itself (oracle/_ref/libchunktrain_ref.so)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO)
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_cache_filled.restype = C.c_int64
            L.ref_tier_log_size.restype = C.c_int64
            cls._lib = L
        return cls._lib

    def __init__(self, cfg: Cfg, real_bytes: int = 4):
        self.L = self.lib()
        self.cfg = cfg
        self.real_bytes = real_bytes
        self.dtype = np.dtype(np.float32 if real_bytes == 4 else np.float64)
        self._err = self.L.ref_last_error
        self._rc = _RefCfg(cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.chunk_size,
                           cfg.page_size, cfg.retrieval_budget, cfg.local_window, cfg.score_scale)
        h = C.c_void_p()
        self._chk(self.L.ref_cache_new(real_bytes, C.byref(self._rc), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_cache_free(self.h)
            self.h = None

    def append(self, layer, k, v):
        k, v = self._a(k), self._a(v)
        b, e = C.c_int64(), C.c_int64()
        self._chk(self.L.ref_cache_append(self.h, layer, _p(k), _p(v), C.c_int64(k.shape[0]), C.byref(b),
                                          C.byref(e)))
        return b.value, e.value

    def n_pages(self, layer):
        return self.L.ref_cache_n_pages(self.h, layer)

    def filled(self, layer):
        return self.L.ref_cache_filled(self.h, layer)

    def page_table(self, layer):
        n = max(self.n_pages(layer), 0)
        out = np.zeros((n, 4), np.int32)
        self._chk(self.L.ref_cache_page_table(self.h, layer, _p(out)))
        return out

    def kavg_raw(self, layer):
        n = self.n_pages(layer)
        s = np.zeros((n, self.cfg.n_kv_heads, self.cfg.head_dim), self.dtype)
        cnt = np.zeros(n, np.int32)
        self._chk(self.L.ref_cache_kavg_raw(self.h, layer, _p(s), _p(cnt)))
        return s, cnt

    def mean_keys(self, layer, n=-1):
        cap = max(self.n_pages(layer), 0)
        out = np.zeros((cap, self.cfg.n_kv_heads, self.cfg.head_dim), self.dtype)
        no = C.c_int()
        self._chk(self.L.ref_cache_mean_keys(self.h, layer, n, _p(out), C.byref(no)))
        return out[: no.value]

    def gather(self, layer, ids, grads=False):
        ids = _i32(ids)
        rows = len(ids) * self.cfg.page_size
        k = np.zeros((rows, self.cfg.n_kv_heads, self.cfg.head_dim), self.dtype)
        v = np.zeros_like(k)
        valid = np.zeros(max(rows, 1), np.uint8)
        self._chk(self.L.ref_cache_gather(self.h, layer, _p(ids), len(ids), int(grads), _p(k), _p(v), _p(valid)))
        return k, v, valid[:rows]

    def scatter(self, layer, ids, dk, dv):
        ids = _i32(ids)
        self._chk(self.L.ref_cache_scatter(self.h, layer, _p(ids), len(ids), _p(self._a(dk)), _p(self._a(dv))))

    def reset(self):
        self._chk(self.L.ref_cache_reset(self.h))

    def zero_grad(self):
        self._chk(self.L.ref_cache_zero_grad(self.h))

    def set_tier(self, layer, page, tier):
        self._chk(self.L.ref_cache_set_tier(self.h, layer, page, tier))

    def set_residency_enforced(self, on):
        self._chk(self.L.ref_cache_set_residency_enforced(self.h, int(on)))

    def memory_report(self) -> dict:
        out = np.zeros(8, np.uint64)
        self._chk(self.L.ref_cache_memory_report(self.h, _p(out)))
        return _report(out)

    def score_pages(self, q, k_avg, score_scale=None):
        q, k_avg = self._a(q), self._a(k_avg)
        cfg = self.cfg
        m = (q.shape[0] + cfg.page_size - 1) // cfg.page_size
        out = np.zeros((m, k_avg.shape[0]), self.dtype)
        sc = cfg.score_scale if score_scale is None else int(score_scale)
        self._chk(self.L.ref_score_pages(self.real_bytes, _p(q), C.c_int64(q.shape[0]), q.shape[1], q.shape[2],
                                         _p(k_avg), C.c_int64(k_avg.shape[0]), k_avg.shape[1], cfg.page_size,
                                         q.shape[1] // k_avg.shape[1], sc, _p(out)))
        return out

    def attn_forward(self, layer, q, selected, k_cur, v_cur):
        q, k_cur, v_cur = self._a(q), self._a(k_cur), self._a(v_cur)
        off, ids = csr(selected)
        out = np.zeros_like(q)
        lse = np.zeros(q.shape[:2], self.dtype)
        self._chk(self.L.ref_attn_forward(self.h, layer, _p(q), C.c_int64(q.shape[0]), _p(off), _p(ids),
                                          C.c_int64(len(selected)), _p(k_cur), _p(v_cur), _p(out), _p(lse)))
        return out, lse

    def attn_backward(self, layer, dout, q, selected, k_cur, v_cur, out, lse):
        dout, q, k_cur, v_cur, out, lse = map(self._a, (dout, q, k_cur, v_cur, out, lse))
        off, ids = csr(selected)
        dq = np.zeros_like(q)
        dk = np.zeros_like(k_cur)
        dv = np.zeros_like(v_cur)
        self._chk(self.L.ref_attn_backward(self.h, layer, _p(dout), _p(q), C.c_int64(q.shape[0]), _p(off),
                                           _p(ids), C.c_int64(len(selected)), _p(k_cur), _p(v_cur), _p(out),
                                           _p(lse), _p(dq), _p(dk), _p(dv)))
        return dq, dk, dv

    def naive_attention(self, q, k, v, past_len, dout, gqa_group):
        q, k, v, dout = map(self._a, (q, k, v, dout))
        out, dq = np.zeros_like(q), np.zeros_like(q)
        dk, dv = np.zeros_like(k), np.zeros_like(v)
        self._chk(self.L.ref_naive_attention(self.real_bytes, _p(q), C.c_int64(q.shape[0]), q.shape[1], q.shape[2],
                                             _p(k), _p(v), C.c_int64(k.shape[0]), k.shape[1], C.c_int64(past_len),
                                             _p(dout), gqa_group, _p(out), _p(dq), _p(dk), _p(dv)))
        return out, dq, dk, dv

    @classmethod
    def select_topk(cls, row, budget) -> np.ndarray:
        L = cls.lib()
        row = np.ascontiguousarray(np.asarray(row, dtype=np.float64))
        out = np.zeros(max(len(row), 1), np.int32)
        cnt = C.c_int()
        rc = L.ref_select_topk(_p(row), len(row), int(budget), _p(out), C.byref(cnt))
        if rc:
            raise OracleError(rc, L.ref_last_error().decode())
        return out[: cnt.value]

    @classmethod
    def select_recent(cls, n_pages, window) -> np.ndarray:
        L = cls.lib()
        out = np.zeros(max(n_pages, 1), np.int32)
        cnt = C.c_int()
        rc = L.ref_select_recent(n_pages, window, _p(out), C.byref(cnt))
        if rc:
            raise OracleError(rc, L.ref_last_error().decode())
        return out[: cnt.value]


class Rng:
    """xoshiro256++ seeded through splitmix64 with Box-Muller normals — the
    reference's bit-stable RNG (common.hpp:31-108), so CPU and GPU harnesses
    share input streams."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        sm = seed & self.M
        self.s = []
        for _ in range(4):
            sm = (sm + 0x9E3779B97F4A7C15) & self.M
            z = sm
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
            self.s.append(z ^ (z >> 31))
        self.spare = None

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & Rng.M

    def next_u64(self) -> int:
        s = self.s
        result = (self._rotl((s[0] + s[3]) & self.M, 23) + s[0]) & self.M
        t = (s[1] << 17) & self.M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def normal(self) -> float:
        import math
        if self.spare is not None:
            v, self.spare = self.spare, None
            return v
        u1 = 0.0
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        theta = 2.0 * 3.14159265358979323846 * u2
        self.spare = r * math.sin(theta)
        return r * math.cos(theta)

    def below(self, n: int) -> int:
        limit = self.M - self.M % n
        while True:
            x = self.next_u64()
            if x < limit:
                return x % n

    def randn(self, *shape, dtype=np.float32) -> np.ndarray:
        n = int(np.prod(shape))
        return np.array([self.normal() for _ in range(n)], dtype=np.float64).astype(dtype).reshape(shape)


def det_normal(seed: int, shape, dtype=np.float32) -> np.ndarray:
    """Version-independent N(0,1) stream: splitmix64 of a counter -> two 53-bit
    uniforms -> Box-Muller. Used for golden-vector inputs so fixtures can store a
    seed instead of the arrays."""
    n = int(np.prod(shape)) if len(shape) else 1
    half = (n + 1) // 2
    with np.errstate(over="ignore"):
        idx = np.arange(2 * half, dtype=np.uint64) + np.uint64((seed & 0xFFFFFFFF) << 32)
        z = idx + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    u1 = np.maximum(u[0::2], 2.0 ** -60)
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(2 * half, np.float64)
    out[0::2] = r * np.cos(2 * np.pi * u2)
    out[1::2] = r * np.sin(2 * np.pi * u2)
    return out[:n].astype(dtype).reshape(shape)


def to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 -> float32 (exact up-cast)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    rounded = (a + np.uint64(0x7FFF) + ((a >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return rounded.astype(np.uint32).view(np.float32).reshape(np.shape(x))


# ---------------------------------------------------------------------------
# Whole-model chunked training step: the reference's
# ChunkTrainer::train_step through the shim. TEST INFRASTRUCTURE.
# ---------------------------------------------------------------------------
class RefModelCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_layers", "d_model", "n_q_heads", "n_kv_heads", "head_dim", "d_ff",
                                       "vocab_size", "chunk_size", "page_size", "retrieval_budget", "local_window",
                                       "score_scale", "mode")] + [("rope_base", C.c_double), ("seed", C.c_uint64)]


MODES = {"dense": 0, "topk": 1, "local": 2}


def ref_model_cfg(mc, mode: str) -> RefModelCfg:
    """chunktrain::ModelConfig fields from a paper_2602_02108_b200 ModelConfig (one mode for all layers)."""
    return RefModelCfg(mc.n_layers, mc.d_model, mc.n_q_heads, mc.n_kv_heads, mc.head_dim, mc.d_ff, mc.vocab_size,
                       mc.chunk_size, mc.page_size, mc.retrieval_budget, mc.local_window, int(mc.score_scale),
                       MODES[mode], mc.rope_base, mc.seed)


def _ref_model_lib():
    L = C.CDLL(build_ref())
    L.ref_model_numel.restype = C.c_int64
    L.ref_last_error.restype = C.c_char_p
    return L


def ref_init_params(mc, mode: str, seed: int, real_bytes: int = 4) -> np.ndarray:
    """init_params (model.hpp:127-145), flattened in ModelParams::visit order."""
    L = _ref_model_lib()
    c = ref_model_cfg(mc, mode)
    n = L.ref_model_numel(C.byref(c))
    out = np.zeros(n, np.float32 if real_bytes == 4 else np.float64)
    if L.ref_init_params(real_bytes, C.byref(c), C.c_uint64(seed), out.ctypes.data_as(C.c_void_p)):
        raise OracleError(9, L.ref_last_error().decode())
    return out


def ref_train_step(mc, mode: str, params: np.ndarray, tokens: np.ndarray):
    """ChunkTrainer<Real>::train_step (chunk_trainer.hpp:131-186) -> (loss, flat grads, selected-id counts
    per (chunk, layer, query page)). Real follows params.dtype."""
    L = _ref_model_lib()
    c = ref_model_cfg(mc, mode)
    rb = params.dtype.itemsize
    params = np.ascontiguousarray(params)
    toks = np.ascontiguousarray(tokens, dtype=np.int32)
    grads = np.zeros_like(params)
    loss = C.c_double()
    n_chunks = (len(toks) + mc.chunk_size - 1) // mc.chunk_size
    counts = np.zeros(n_chunks * mc.n_layers * (mc.chunk_size // mc.page_size), np.int32)
    rc = L.ref_train_step(rb, C.byref(c), params.ctypes.data_as(C.c_void_p), toks.ctypes.data_as(C.c_void_p),
                          C.c_int64(len(toks)), grads.ctypes.data_as(C.c_void_p), C.byref(loss),
                          counts.ctypes.data_as(C.c_void_p))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return loss.value, grads, counts


def ref_full_forward_backward(mc, params: np.ndarray, tokens: np.ndarray):
    """full_forward_backward (oracle.hpp:89-276): the non-chunked ground truth -> (loss, flat grads)."""
    L = _ref_model_lib()
    c = ref_model_cfg(mc, "dense")
    params = np.ascontiguousarray(params)
    toks = np.ascontiguousarray(tokens, dtype=np.int32)
    grads = np.zeros_like(params)
    loss = C.c_double()
    rc = L.ref_full_forward_backward(params.dtype.itemsize, C.byref(c), params.ctypes.data_as(C.c_void_p),
                                     toks.ctypes.data_as(C.c_void_p), C.c_int64(len(toks)),
                                     grads.ctypes.data_as(C.c_void_p), C.byref(loss))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return loss.value, grads


class RefTierCfgC(C.Structure):
    _fields_ = [("device_capacity_pages", C.c_int64), ("bandwidth_bytes_per_s", C.c_double),
                ("fixed_s_per_layer", C.c_double), ("s_per_attended_token", C.c_double)]


def ref_train_step_offload(mc, mode: str, params: np.ndarray, tokens: np.ndarray, capacity: int,
                           bandwidth: float = 16e9, fixed_s: float = 1e-3, s_per_token: float = 1e-6):
    """ChunkTrainer::train_step with enable_offload (chunk_trainer.hpp:118-186) -> (loss, flat grads,
    ScheduleLog events as an int64 array [n, 6] of (kind, layer, page, chunk, phase, bytes) plus times)."""
    L = _ref_model_lib()
    c = ref_model_cfg(mc, mode)
    tc = RefTierCfgC(capacity, bandwidth, fixed_s, s_per_token)
    params = np.ascontiguousarray(params)
    toks = np.ascontiguousarray(tokens, dtype=np.int32)
    grads = np.zeros_like(params)
    loss = C.c_double()
    cap = 1 << 16
    evs = (RefEvent * cap)()
    n = C.c_int64()
    rc = L.ref_train_step_offload(params.dtype.itemsize, C.byref(c), params.ctypes.data_as(C.c_void_p),
                                  toks.ctypes.data_as(C.c_void_p), C.c_int64(len(toks)), C.byref(tc),
                                  grads.ctypes.data_as(C.c_void_p), C.byref(loss), evs, C.c_int64(cap), C.byref(n))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    ev = np.array([(e.kind, e.layer, e.page, e.chunk, e.phase, e.bytes) for e in evs[: n.value]], np.int64)
    t = np.array([e.t for e in evs[: n.value]])
    return loss.value, grads, ev, t
