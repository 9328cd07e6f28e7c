// SPDX-License-Identifier: Apache-2.0
//
// chunktrain/attention.hpp — the reference's attention operators (attention.hpp:32-293) with
// their host signatures, computed on the B200 by liboomb.so (score_pages, select_topk(_row),
// select_recent / select_all, attn_forward, attn_backward). Source-compatibility header: see
// chunktrain/common.hpp. Real = float runs the fp32 device path, Real = double the fp64 one.
#pragma once

#include <span>
#include <utility>
#include <vector>

#include "chunktrain/paged_kv.hpp"

namespace chunktrain {

// (parameters are chunktrain::Tensor so these overloads are exact matches: the facade's own
// oomb:: overloads, reachable by argument-dependent lookup through the base class, need a
// derived-to-base conversion and lose)
template <class Real>
Tensor<Real> score_pages(const Tensor<Real>& q, const Tensor<Real>& k_avg, int page_size, int gqa_group,
                         bool score_scale = false) {
    return oomb::score_pages(q, k_avg, page_size, gqa_group, score_scale);
}

inline std::vector<int32_t> select_topk(std::span<const double> score_row, int budget_pages) {
    return oomb::select_topk(score_row, budget_pages);
}
inline std::vector<int32_t> select_topk(const std::vector<double>& score_row, int budget_pages) {
    return oomb::select_topk(std::span<const double>(score_row), budget_pages);
}
template <class Real>
std::vector<int32_t> select_topk_row(const Tensor<Real>& score, int64_t row, int budget_pages) {
    return oomb::select_topk_row(score, row, budget_pages);
}
using oomb::select_all;
using oomb::select_recent;

template <class Real>
struct AttnSaved {  // attention.hpp:117-124
    Tensor<Real> out;
    Tensor<Real> lse;
    std::vector<std::vector<int32_t>> selected;
};
template <class Real>
struct AttnGrads {  // attention.hpp:210-220
    Tensor<Real> dq;
    Tensor<Real> dk_cur;
    Tensor<Real> dv_cur;
};

template <class Real>
AttnSaved<Real> attn_forward(const ModelConfig& cfg, const oomb::Tensor<Real>& q, PagedCache<Real>& cache, int layer,
                             std::vector<std::vector<int32_t>> selected, const oomb::Tensor<Real>& k_cur,
                             const oomb::Tensor<Real>& v_cur) {
    auto s = oomb::attn_forward(cfg, q, cache.device(), layer, std::move(selected), k_cur, v_cur);
    return AttnSaved<Real>{std::move(s.out), std::move(s.lse), std::move(s.selected)};
}

template <class Real>
AttnGrads<Real> attn_backward(const ModelConfig& cfg, const oomb::Tensor<Real>& dout, const oomb::Tensor<Real>& q,
                              PagedCache<Real>& cache, int layer, const oomb::Tensor<Real>& k_cur,
                              const oomb::Tensor<Real>& v_cur, const AttnSaved<Real>& saved) {
    const oomb::AttnSaved<Real> s{saved.out, saved.lse, saved.selected};
    auto g = oomb::attn_backward(cfg, dout, q, cache.device(), layer, k_cur, v_cur, s);
    return AttnGrads<Real>{std::move(g.dq), std::move(g.dk_cur), std::move(g.dv_cur)};
}

}  // namespace chunktrain
