"""CPU-only checks of the drop-in boundary: liboomb.so loads without a GPU,
exports every symbol include/oomb.h declares, and its host logic (the page
table mirror of PagedCache and ModelConfig validation) matches the reference."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle.oracle import Cfg, Port, Ref, det_normal
from paper_2602_02108_b200 import ConfigError, ModelConfig, parse_model_config
from paper_2602_02108_b200 import _lib
from paper_2602_02108_b200._lib import OombMemoryReport, call

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "oomb.h")).read()
    return sorted(set(re.findall(r"^OOMB_API\s+[\w\s\*]+?\b(oomb_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.exported_symbols())
    assert L.oomb_version() == 1


def test_comm_library_exports_every_header_symbol():
    """liboomb_comm.so (NCCL exchange steps) loads without a GPU and exports include/oomb_comm.h."""
    src = open(os.path.join(ROOT, "include", "oomb_comm.h")).read()
    syms = sorted(set(re.findall(r"^OOMB_API\s+[\w\s\*]+?\b(oomb_\w+)\s*\(", src, flags=re.M)))
    assert len(syms) == 11
    L = _lib.comm_lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.comm_exported_symbols())
    # argument checks happen before any NCCL / CUDA call
    from paper_2602_02108_b200 import errors
    with pytest.raises(errors.ConfigError):
        _lib.comm_call("oomb_comm_init", (C.c_uint8 * 128)(), 3, 2, 0, C.byref(C.c_void_p()))
    with pytest.raises(errors.StateError):
        _lib.comm_call("oomb_dq_reduce", None, None, 4, None, None)


def test_library_carries_sm100a_tensor_core_code():
    import subprocess
    so = _lib.LIB_PATH
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass      # tcgen05.mma
    assert "UTMALDG" in sass      # TMA tile loads
    assert "LDTM" in sass         # tcgen05.ld
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", so], capture_output=True,
                                       text=True).stdout


class PT:
    """Thin wrapper over oomb_pagetable_* (no device)."""

    def __init__(self, cfg: Cfg, kv_elem=4, grad_elem=4):
        h = C.c_void_p()
        call("oomb_pagetable_create", cfg.n_layers, cfg.page_size, cfg.n_kv_heads, cfg.head_dim, kv_elem, grad_elem,
             C.byref(h))
        self.h = h
        self.cfg = cfg

    def __del__(self):
        _lib.lib().oomb_pagetable_destroy(self.h)

    def append(self, layer, rows):
        b, e = C.c_int64(), C.c_int64()
        call("oomb_pagetable_append", self.h, layer, rows, C.byref(b), C.byref(e))
        return b.value, e.value

    def scatter(self, layer, ids):
        ids = np.ascontiguousarray(np.asarray(ids, np.int32))
        call("oomb_pagetable_scatter", self.h, layer, ids.ctypes.data_as(C.c_void_p), len(ids))

    def reset(self):
        call("oomb_pagetable_reset", self.h)

    def n_pages(self, layer):
        n = C.c_int()
        call("oomb_pagetable_n_pages", self.h, layer, C.byref(n))
        return n.value

    def table(self, layer):
        n = self.n_pages(layer)
        out = np.zeros((max(n, 1), 4), np.int32)
        call("oomb_pagetable_get", self.h, layer, out.ctypes.data_as(C.c_void_p))
        return out[:n]

    def report(self):
        r = OombMemoryReport()
        call("oomb_pagetable_memory_report", self.h, C.byref(r))
        return r


def run_script(backend, seed, steps=4):
    """Random append/scatter/reset script; returns page tables + reports per step."""
    rng = np.random.default_rng(seed)
    cfg = backend.cfg
    snaps = []
    for step in range(steps):
        for layer in range(cfg.n_layers):
            for _ in range(int(rng.integers(1, 5))):
                rows = int(rng.integers(0, 3 * cfg.page_size))
                if isinstance(backend, PT):
                    backend.append(layer, rows)
                else:
                    z = np.zeros((rows, cfg.n_kv_heads, cfg.head_dim), backend.dtype)
                    backend.append(layer, z, z)
            n = backend.n_pages(layer)
            if n:
                ids = rng.permutation(n)[: max(1, n // 2)].astype(np.int32)
                if isinstance(backend, PT):
                    backend.scatter(layer, ids)
                else:
                    g = np.zeros((len(ids) * cfg.page_size, cfg.n_kv_heads, cfg.head_dim), backend.dtype)
                    backend.scatter(layer, ids, g, g)
        tabs = [backend.table(l) if isinstance(backend, PT) else backend.page_table(l) for l in range(cfg.n_layers)]
        if isinstance(backend, PT):
            r = backend.report()
            rep = (r.device_bytes, r.grad_bytes, r.pages, r.arena_blocks, r.free_list)
        else:
            r = backend.memory_report()
            rep = (r["device_bytes"], r["grad_bytes"], r["pages"], r["arena_blocks"], r["free_list"])
        snaps.append((tabs, rep))
        backend.reset()
    return snaps


@pytest.mark.parametrize("seed", range(6))
def test_pagetable_host_logic_matches_reference(seed):
    cfg = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16, retrieval_budget=32)
    ref = Ref(cfg, 4) if Ref.available() else Port(cfg, 4)
    a = run_script(PT(cfg), seed)
    b = run_script(ref, seed)
    for (ta, ra), (tb, rb) in zip(a, b):
        for x, y in zip(ta, tb):
            assert x.tolist() == y.tolist()
        assert ra == rb


def test_pagetable_golden_script_tables():
    """The golden pagetable script's tables (made by the reference) are reproduced."""
    g = np.load(os.path.join(G, "pagetable.npz"))
    cfg = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16, retrieval_budget=32)
    pt = PT(cfg)
    rng = np.random.default_rng(5)
    for step in range(3):
        for layer in range(2):
            for _ in range(int(rng.integers(1, 5))):
                rows = int(rng.integers(1, 40))
                pt.append(layer, rows)
            n = pt.n_pages(layer)
            ids = sorted(set(int(x) for x in rng.integers(0, n, size=max(1, n // 2))))
            rng.shuffle(ids)
            pt.scatter(layer, ids)
        for layer in range(2):
            assert pt.table(layer).tolist() == g[f"s{step}/pt{layer}"].tolist()
        r = pt.report()
        want = g[f"s{step}/report"]
        assert [r.device_bytes, r.host_bytes, r.grad_bytes, r.pages, r.arena_blocks, r.free_list] == want.tolist()
        pt.reset()


def test_pagetable_reference_known_answers():
    """test_paged_kv.cpp:57-97,221-269 arithmetic on the host mirror."""
    cfg = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=128,
              retrieval_budget=256)
    pt = PT(cfg)
    assert pt.append(0, 130) == (0, 130)
    assert pt.n_pages(0) == 2
    pt2 = PT(cfg)
    pt2.append(1, 64)
    pt2.append(1, 64)
    assert pt2.n_pages(1) == 1
    c16 = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16, retrieval_budget=32)
    p3 = PT(c16)
    for l in range(2):
        p3.append(l, 3 * 16)
    r = p3.report()
    assert (r.pages, r.device_bytes, r.grad_bytes) == (6, 24576, 0)
    blocks = r.arena_blocks
    p3.reset()
    assert p3.report().free_list == blocks
    for l in range(2):
        p3.append(l, 2 * 16)
    assert p3.report().arena_blocks == blocks
    with pytest.raises(Exception):
        p3.append(5, 4)


def test_model_config_validation_and_parser():
    ModelConfig().validate()
    with pytest.raises(ConfigError):
        ModelConfig(n_q_heads=3, n_kv_heads=2).validate()
    with pytest.raises(ConfigError):
        ModelConfig(chunk_size=100, page_size=16).validate()
    with pytest.raises(ConfigError):
        ModelConfig(head_dim=7).validate()
    cfg = parse_model_config("n_layers = 1\nn_q_heads=28\nn_kv_heads = 4 # qwen\nhead_dim=128\n"
                             "chunk_size=4096\npage_size=128\nretrieval_budget=8192\nattention_mode=topk\n")
    assert cfg.budget_pages() == 64 and cfg.gqa_group() == 7 and cfg.mode_for_layer(0) == "topk"
    with pytest.raises(ConfigError):
        parse_model_config("bogus = 1\n")
