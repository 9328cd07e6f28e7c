// SPDX-License-Identifier: Apache-2.0
//
// chunktrain/oracle.hpp — TEST INFRASTRUCTURE. The reference tests' monolithic checker
// naive_attention_fwd_bwd (oracle.hpp:285-360) mapped onto this repository's CPU oracle
// (oracle/oomb_oracle.c, oc_naive_attention_*): link liboomb_oracle.so. Never part of the product
// path; only the reference's own test sources include it (source-compatibility: see
// chunktrain/common.hpp).
#pragma once

#include <type_traits>

#include "chunktrain/tensor.hpp"

extern "C" {
int oc_naive_attention_f32(const float* q, int64_t tq, int qh, int hd, const float* k, const float* v, int64_t tk,
                           int kvh, int64_t past_len, const float* dout, int gqa_group, float* out, float* dq,
                           float* dk, float* dv);
int oc_naive_attention_f64(const double* q, int64_t tq, int qh, int hd, const double* k, const double* v, int64_t tk,
                           int kvh, int64_t past_len, const double* dout, int gqa_group, double* out, double* dq,
                           double* dk, double* dv);
}

namespace chunktrain {

template <class Real>
struct NaiveAttnResult {
    Tensor<Real> out, dq, dk, dv;
};

template <class Real>
NaiveAttnResult<Real> naive_attention_fwd_bwd(const oomb::Tensor<Real>& q, const oomb::Tensor<Real>& k,
                                              const oomb::Tensor<Real>& v, int64_t past_len,
                                              const oomb::Tensor<Real>& dout, int gqa_group) {
    static_assert(std::is_same_v<Real, float> || std::is_same_v<Real, double>, "float or double");
    NaiveAttnResult<Real> r{Tensor<Real>(q.shape), Tensor<Real>(q.shape), Tensor<Real>(k.shape), Tensor<Real>(k.shape)};
    int rc;
    if constexpr (std::is_same_v<Real, float>)
        rc = oc_naive_attention_f32(q.data.data(), q.dim(0), static_cast<int>(q.dim(1)), static_cast<int>(q.dim(2)),
                                    k.data.data(), v.data.data(), k.dim(0), static_cast<int>(k.dim(1)), past_len,
                                    dout.data.data(), gqa_group, r.out.ptr(), r.dq.ptr(), r.dk.ptr(), r.dv.ptr());
    else
        rc = oc_naive_attention_f64(q.data.data(), q.dim(0), static_cast<int>(q.dim(1)), static_cast<int>(q.dim(2)),
                                    k.data.data(), v.data.data(), k.dim(0), static_cast<int>(k.dim(1)), past_len,
                                    dout.data.data(), gqa_group, r.out.ptr(), r.dq.ptr(), r.dk.ptr(), r.dv.ptr());
    if (rc) throw ShapeError("naive_attention_fwd_bwd: oracle error");
    return r;
}

}  // namespace chunktrain
