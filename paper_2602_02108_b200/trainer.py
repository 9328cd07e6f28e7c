"""Whole-model chunk-recurrent training step on the device.

ChunkTrainer::train_step (chunk_trainer.hpp:131-186): phase A runs every chunk forward in order
(append K/V, select pages, attend; activations are dropped), then every chunk in reverse order
recomputes its forward with an activation tape and back-propagates. Gradients reach earlier
chunks only through the paged gradient pool: attn_backward adds past-page dK/dV into it, and each
chunk reads back its own pages' gradients (dM_i, chunk_trainer.hpp:575-587) before the K/V
projections.

The hot path is the library's (paged attention fwd/bwd, page selection, append, RoPE, grad
pages). The rest of the model (RMSNorm, projections, SiLU MLP, cross entropy) is plain fp32
torch on the device: cuBLAS GEMMs (TF32 off) and elementwise ops, each restating ops.hpp.
Parameters use the reference layouts (`y = x @ W`, W [in x out]) and ModelParams::visit order
(model.hpp:66-81), so a parameter vector moves between the two implementations unchanged.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import attention as A
from .config import ModelConfig
from .errors import StateError
from .paged_kv import PagedCache
from .tiered_memory import BACKWARD, FORWARD, ComputeCostModel, TierConfig, TieredEngine

RMS_EPS = 1e-6        # kRmsNormEps, chunk_trainer.hpp:31
IGNORE_TARGET = -1    # kIgnoreTarget, ops.hpp:268

LAYER_PARAMS = ("wq", "wk", "wv", "wo", "w_up", "w_down", "attn_norm", "mlp_norm")


def param_shapes(cfg: ModelConfig) -> list[tuple[str, int, tuple[int, ...]]]:
    """(name, layer, shape) in ModelParams::visit order (model.hpp:66-81); layer -1 = global."""
    d, qd, kd = cfg.d_model, cfg.n_q_heads * cfg.head_dim, cfg.n_kv_heads * cfg.head_dim
    out = [("emb", -1, (cfg.vocab_size, d)), ("unemb", -1, (d, cfg.vocab_size)), ("final_norm", -1, (d,))]
    per = {"wq": (d, qd), "wk": (d, kd), "wv": (d, kd), "wo": (qd, d), "w_up": (d, cfg.d_ff),
           "w_down": (cfg.d_ff, d), "attn_norm": (d,), "mlp_norm": (d,)}
    for l in range(cfg.n_layers):
        out += [(n, l, per[n]) for n in LAYER_PARAMS]
    return out


def unflatten(flat, cfg: ModelConfig, device) -> dict:
    """Flat parameter vector (visit order) -> {"emb": T, ..., "layers": [{"wq": T, ...}, ...]}."""
    flat = torch.as_tensor(np.asarray(flat, dtype=np.float32)).to(device)
    p: dict = {"layers": [dict() for _ in range(cfg.n_layers)]}
    o = 0
    for name, layer, shape in param_shapes(cfg):
        n = int(np.prod(shape))
        t = flat[o:o + n].view(shape).clone()
        o += n
        (p if layer < 0 else p["layers"][layer])[name] = t
    if o != flat.numel():
        raise ValueError("parameter vector does not match the configuration")
    return p


def flatten(p: dict, cfg: ModelConfig) -> torch.Tensor:
    return torch.cat([(p if layer < 0 else p["layers"][layer])[name].reshape(-1)
                      for name, layer, _ in param_shapes(cfg)])


def zeros_like(p: dict) -> dict:
    return {k: ([{n: torch.zeros_like(t) for n, t in l.items()} for l in v] if k == "layers" else torch.zeros_like(v))
            for k, v in p.items()}


# ---------------------------------------------------------------------------- ops.hpp restated
def rmsnorm(x, g):  # ops.hpp:132-149
    inv = torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + RMS_EPS)
    return x * inv * g


def rmsnorm_backward(x, g, dy, dg_accum):  # ops.hpp:151-183
    d = x.shape[-1]
    inv = torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + RMS_EPS)
    dg_accum += (dy * x * inv).sum(dim=0)
    dot = (dy * g * x).sum(dim=-1, keepdim=True)
    return dy * g * inv - x * (inv * inv * inv * dot / d)


def silu(x):  # ops.hpp:236-244
    return x * torch.sigmoid(x)


def silu_backward(x, dy):  # ops.hpp:246-256
    s = torch.sigmoid(x)
    return dy * s * (1 + x * (1 - s))


def linear_backward(x, w, dy, dw_accum):  # ops.hpp:46-86: dX = dY W^T, dW += x^T dY
    dw_accum += x.t() @ dy
    return dy @ w.t()


def cross_entropy_scaled(logits, targets, scale: float):  # ops.hpp:273-306
    """(sum of the per-row NLL over rows with a target, dlogits = (softmax - onehot) * scale)."""
    keep = targets != IGNORE_TARGET
    lse = torch.logsumexp(logits, dim=-1)
    tg = targets.clamp(min=0)
    nll = (lse - logits.gather(1, tg[:, None])[:, 0]) * keep
    d = torch.softmax(logits, dim=-1) * scale
    d[torch.arange(len(tg), device=logits.device), tg] -= scale
    d *= keep[:, None]
    return float(nll.sum()), d


# ---------------------------------------------------------------------------- the chunk loop
@dataclass
class ChunkState:  # chunk_trainer.hpp:36-48
    index: int
    pos_offset: int
    tokens: torch.Tensor           # [C] int64, device
    targets: torch.Tensor          # [C] int64, device (IGNORE_TARGET where none)
    selected: list                 # per layer: Selection


@dataclass
class StepMetrics:
    loss: float


class ChunkTrainer:
    """Device counterpart of chunktrain::ChunkTrainer<float> for one sequence. With a TierConfig
    (enable_offload, chunk_trainer.hpp:118-124) every step runs the reference's residency protocol
    on a TieredEngine: lookahead prefetch, ensure_resident_, end_layer_use, grads-scattered marks and
    the cost-model clock (chunk_trainer.hpp:318-363, 388-462, 531-541), with real page moves."""

    def __init__(self, cfg: ModelConfig, max_tokens: int, dtype: str = "fp32", tier: TierConfig | None = None):
        cfg.validate()
        self.cfg = cfg
        self.cache = PagedCache(cfg, dtype=dtype, max_tokens=max_tokens)
        self.dev = self.cache.device
        self.dtype = self.cache.dtype
        self.chunks: list[ChunkState] = []
        self.tier = tier
        self.engine: TieredEngine | None = None
        self.pending = None
        self.last_log = None  # raw ScheduleLog events of the last offloaded step

    def enable_offload(self, tier: TierConfig) -> None:
        self.tier = tier

    def disable_offload(self) -> None:
        self.tier = None

    # ---- residency protocol (chunk_trainer.hpp:318-363)
    @staticmethod
    def _union(sel) -> list[int]:
        return sorted({int(p) for l in sel.lists() for p in l})

    def _attended(self, sel) -> int:  # attended_tokens_ (chunk_trainer.hpp:318-322)
        return self.cfg.chunk_size + sum(len(l) for l in sel.lists()) * self.cfg.page_size

    def _lookahead(self, nxt: ChunkState, layer: int, cached: bool, backward_part: bool) -> None:
        eng, cfg = self.engine, self.cfg
        if eng is None:
            return
        if cached:
            pages = self._union(nxt.selected[layer])
            if backward_part:
                pages = sorted(set(pages) | set(self._own_pages(nxt).tolist()))
        else:
            mode = cfg.mode_for_layer(layer)
            if mode == "topk":
                return  # sparse ids appear only after that layer's q projection
            n_cand = nxt.pos_offset // cfg.page_size
            pages = A.select_all(n_cand) if mode == "dense" else A.select_recent(n_cand, cfg.local_window)
            existing = self.cache.n_pages(layer)
            pages = [p for p in pages if p < existing]  # pages appended later are device-born
        self.pending = eng.fetch_async(layer, pages, nxt.index, best_effort=True)

    def _ensure_resident(self, layer: int, ids, chunk_idx: int, h_cur) -> None:
        eng = self.engine
        if eng is None:
            return
        if h_cur is not None:
            eng.wait(h_cur)
        eng.wait(eng.fetch_async(layer, ids, chunk_idx))
        eng.record_access(layer, ids, chunk_idx)

    def _cost(self) -> ComputeCostModel:
        return self.tier.compute

    def make_chunk_states(self, tokens) -> list[ChunkState]:  # chunk_trainer.hpp:225-251
        toks = np.asarray(tokens, dtype=np.int64)
        t_total, c = len(toks), self.cfg.chunk_size
        out = []
        for i in range((t_total + c - 1) // c):
            pos = i * c
            tk = np.zeros(c, np.int64)
            tg = np.full(c, IGNORE_TARGET, np.int64)
            n = min(c, t_total - pos)
            tk[:n] = toks[pos:pos + n]
            m = max(0, min(c, t_total - pos - 1))
            tg[:m] = toks[pos + 1:pos + 1 + m]
            out.append(ChunkState(i, pos, torch.from_numpy(tk).to(self.dev), torch.from_numpy(tg).to(self.dev), []))
        return out

    # ---- selection (chunk_trainer.hpp:292-316)
    def _select(self, chunk: ChunkState, layer: int, q_rope) -> A.Selection:
        cfg = self.cfg
        m = cfg.pages_per_chunk()
        n_cand = chunk.pos_offset // cfg.page_size
        mode = cfg.mode_for_layer(layer)
        if n_cand == 0:
            return A.Selection.from_lists(self.cache, [[]] * m)
        if mode == "dense":
            return A.Selection.from_lists(self.cache, [A.select_all(n_cand)] * m)
        if mode == "local":
            return A.Selection.from_lists(self.cache, [A.select_recent(n_cand, cfg.local_window)] * m)
        return A.select_pages_topk(self.cache, layer, q_rope, n_cand)

    def _own_pages(self, chunk: ChunkState) -> np.ndarray:
        m = self.cfg.pages_per_chunk()
        return np.arange(chunk.index * m, (chunk.index + 1) * m, dtype=np.int32)

    def _run_chunk(self, p: dict, chunk: ChunkState, append: bool, tape: list | None, loss_scale: float):
        """chunk_trainer.hpp:388-501: the shared chunk pass; append=True is phase A."""
        cfg, C = self.cfg, self.cfg.chunk_size
        hq, hk, hd = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
        eng = self.engine
        h = p["emb"][chunk.tokens]
        for l in range(cfg.n_layers):
            lp = p["layers"][l]
            h_cur = None
            if eng is not None:  # prefetch for the step that follows this one
                h_cur, self.pending = self.pending, None
                if l + 1 < cfg.n_layers:
                    self._lookahead(chunk, l + 1, cached=not append, backward_part=False)
                elif append:
                    if chunk.index + 1 < len(self.chunks):
                        self._lookahead(self.chunks[chunk.index + 1], 0, cached=False, backward_part=False)
                else:  # last recompute layer: this chunk's backward of the same layer comes next
                    self._lookahead(chunk, l, cached=True, backward_part=True)
            a = rmsnorm(h, lp["attn_norm"])
            q = A.rope((a @ lp["wq"]).view(C, hq, hd), chunk.pos_offset, cfg.rope_base, out_dtype=self.dtype)
            if eng is not None:
                eng.advance_compute(self._cost().q_time(), chunk.index, l)
            if append:
                chunk.selected.append(self._select(chunk, l, q))
                if eng is not None and cfg.mode_for_layer(l) == "topk":
                    h_cur = eng.fetch_async(l, self._union(chunk.selected[l]), chunk.index)
            sel = chunk.selected[l]
            sel_union = self._union(sel) if eng is not None else None
            k = A.rope((a @ lp["wk"]).view(C, hk, hd), chunk.pos_offset, cfg.rope_base, out_dtype=self.dtype)
            v = (a @ lp["wv"]).view(C, hk, hd).to(self.dtype).contiguous()
            if eng is not None:
                eng.advance_compute(self._cost().kv_time(), chunk.index, l)
            if append:
                r = self.cache.append_chunk(l, k, v)
                if eng is not None:
                    eng.on_pages_appended(l, r)
            self._ensure_resident(l, sel_union, chunk.index, h_cur)
            saved = A.attn_forward(cfg, q, self.cache, l, sel, k, v)
            if eng is not None:
                eng.advance_compute(self._cost().attn_time(self._attended(sel)), chunk.index, l)
            attn_flat = saved.out.view(C, hq * hd).float()
            h2 = h + attn_flat @ lp["wo"]
            b = rmsnorm(h2, lp["mlp_norm"])
            u = b @ lp["w_up"]
            s = silu(u)
            h_next = h2 + s @ lp["w_down"]
            if eng is not None:
                eng.advance_compute(self._cost().post_time(), chunk.index, l)
                used = sel_union + (self._own_pages(chunk).tolist() if append else [])
                eng.end_layer_use(l, used)
            if tape is not None:
                tape.append(dict(attn_norm_in=h, a=a, q=q, k=k, v=v, saved=saved, attn_flat=attn_flat, h2=h2, b=b,
                                 u=u, s=s))
            h = h_next
        fn = rmsnorm(h, p["final_norm"])
        logits = fn @ p["unemb"]
        loss, dlogits = cross_entropy_scaled(logits, chunk.targets, loss_scale)
        if not np.isfinite(loss):
            raise StateError("non-finite loss in chunk forward")
        return loss, dlogits, h, fn

    def _backward(self, p: dict, chunk: ChunkState, tape: list, final_in, fn, dlogits, g: dict) -> None:
        """chunk_trainer.hpp:503-614 (backward_from_loss_)."""
        cfg, C = self.cfg, self.cfg.chunk_size
        hq, hk, hd = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
        dfn = linear_backward(fn, p["unemb"], dlogits, g["unemb"])
        dh = rmsnorm_backward(final_in, p["final_norm"], dfn, g["final_norm"])
        own = self._own_pages(chunk)
        eng = self.engine
        for l in reversed(range(cfg.n_layers)):
            lp, lg, la = p["layers"][l], g["layers"][l], tape[l]
            sel = chunk.selected[l]
            h_cur = None
            if eng is not None:
                h_cur, self.pending = self.pending, None
                if l > 0:
                    self._lookahead(chunk, l - 1, cached=True, backward_part=True)
                elif chunk.index > 0:
                    self._lookahead(self.chunks[chunk.index - 1], 0, cached=True, backward_part=False)
                eng.advance_compute(2 * self._cost().post_time(), chunk.index, l)
            ds = linear_backward(la["s"], lp["w_down"], dh, lg["w_down"])
            du = silu_backward(la["u"], ds)
            db = linear_backward(la["b"], lp["w_up"], du, lg["w_up"])
            dh2 = rmsnorm_backward(la["h2"], lp["mlp_norm"], db, lg["mlp_norm"]) + dh
            dattn = linear_backward(la["attn_flat"], lp["wo"], dh2, lg["wo"])
            dout = dattn.view(C, hq, hd).to(self.dtype).contiguous()
            touch = None
            if eng is not None:
                sel_union = self._union(sel)
                touch = sorted(set(sel_union) | set(own.tolist()))
                self._ensure_resident(l, touch, chunk.index, h_cur)
            ag = A.attn_backward(cfg, dout, la["q"], self.cache, l, la["k"], la["v"], la["saved"])
            if eng is not None:
                eng.on_grads_scattered(l, sel_union)
                eng.advance_compute(2 * self._cost().attn_time(self._attended(sel)), chunk.index, l)
            # dM_i: what later chunks deposited into this chunk's own pages joins dK / dV, and dK is
            # rotated back in the same pass (the reverse projection epilogue)
            self.cache.accumulate_grad_pages_rope(l, own, ag.dk_cur, ag.dv_cur, chunk.pos_offset, cfg.rope_base)
            dq_pre = A.rope(ag.dq, chunk.pos_offset, cfg.rope_base, sign=-1).view(C, hq * hd)
            dk_pre = ag.dk_cur.view(C, hk * hd)
            da = linear_backward(la["a"], lp["wq"], dq_pre, lg["wq"])
            da = da + linear_backward(la["a"], lp["wk"], dk_pre, lg["wk"])
            da = da + linear_backward(la["a"], lp["wv"], ag.dv_cur.view(C, hk * hd), lg["wv"])
            dh = rmsnorm_backward(la["attn_norm_in"], lp["attn_norm"], da, lg["attn_norm"]) + dh2
            if eng is not None:
                eng.advance_compute(2 * (self._cost().q_time() + self._cost().kv_time()), chunk.index, l)
                eng.end_layer_use(l, touch)
        # embedding rows (chunk_trainer.hpp:616-621): a one-hot GEMM keeps the sum order fixed (an
        # atomic index_add would make repeated tokens' sums run-to-run different); large vocabularies
        # fall back to index_add
        if cfg.vocab_size * C <= 1 << 24:
            onehot = torch.zeros(C, cfg.vocab_size, device=dh.device, dtype=dh.dtype)
            onehot[torch.arange(C, device=dh.device), chunk.tokens] = 1.0
            g["emb"] += onehot.t() @ dh
        else:
            g["emb"].index_add_(0, chunk.tokens, dh)

    def train_step(self, p: dict, tokens, grads_out: dict | None = None) -> tuple[StepMetrics, dict]:
        """chunk_trainer.hpp:131-186. Returns (metrics, gradients) with the gradients in the same
        structure as the parameters (zeroed first, or accumulated into grads_out after zeroing)."""
        t_total = len(tokens)
        if t_total == 0:
            raise StateError("train_step: empty token sequence")
        g = zeros_like(p) if grads_out is None else grads_out
        if grads_out is not None:
            for k, v in g.items():
                if k == "layers":
                    for l in v:
                        for t in l.values():
                            t.zero_()
                else:
                    v.zero_()
        self.cache.reset()
        self.chunks = self.make_chunk_states(tokens)
        self.pending = None
        self.engine = None
        if self.tier is not None:
            self.engine = TieredEngine(self.cache, self.tier)
            self.engine.set_prefetch_headroom_pages(self.cfg.pages_per_chunk())
            self.engine.begin_phase(FORWARD)
        scale = 1.0 / (t_total - 1) if t_total > 1 else 1.0
        loss_sum = 0.0
        try:
            with torch.no_grad():
                for ch in self.chunks:  # phase A
                    loss_sum += self._run_chunk(p, ch, True, None, 1.0)[0]
                if self.engine is not None:
                    self.engine.release_all_reservations()
                    self.engine.begin_phase(BACKWARD)
                self.pending = None
                if self.engine is not None and self.chunks:  # head start for the first recompute step
                    self._lookahead(self.chunks[-1], 0, cached=True, backward_part=False)
                for ch in reversed(self.chunks):  # recompute + backward, reverse chunk order
                    tape: list = []
                    _, dlogits, final_in, fn = self._run_chunk(p, ch, False, tape, scale)
                    self._backward(p, ch, tape, final_in, fn, dlogits, g)
            if self.engine is not None:
                torch.cuda.synchronize()
                self.last_log = self.engine.raw_log()
        finally:
            if self.engine is not None:
                self.engine.close(discard=True)  # the cache is reset every step (chunk_trainer.hpp:136)
                self.engine = None
        loss = loss_sum / (t_total - 1) if t_total > 1 else 0.0
        return StepMetrics(loss), g
