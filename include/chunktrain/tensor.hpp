// SPDX-License-Identifier: Apache-2.0
//
// chunktrain/tensor.hpp — the reference's host value type (tensor.hpp:19-125 and the error
// metrics :157-170) as the facade's oomb::Tensor<Real> plus the element accessors reference
// call sites use. Source-compatibility header: see chunktrain/common.hpp.
#pragma once

#include <algorithm>
#include <cmath>
#include <initializer_list>

#include "chunktrain/common.hpp"

namespace chunktrain {

template <class Real>
struct Tensor : oomb::Tensor<Real> {
    using Base = oomb::Tensor<Real>;
    using Base::Base;
    Tensor() = default;
    Tensor(const Base& b) : Base(b) {}  // NOLINT: results of facade calls convert implicitly
    Tensor(Base&& b) : Base(std::move(b)) {}  // NOLINT

    size_t bytes() const { return this->data.size() * sizeof(Real); }
    bool same_shape(const oomb::Tensor<Real>& o) const { return this->shape == o.shape; }
    Real* ptr() { return this->data.data(); }
    const Real* ptr() const { return this->data.data(); }
    Real& operator()(int64_t i) { return this->data[static_cast<size_t>(i)]; }
    Real operator()(int64_t i) const { return this->data[static_cast<size_t>(i)]; }
    Real& operator()(int64_t i, int64_t j) { return this->data[static_cast<size_t>(i * this->dim(1) + j)]; }
    Real operator()(int64_t i, int64_t j) const { return this->data[static_cast<size_t>(i * this->dim(1) + j)]; }
    Real& operator()(int64_t i, int64_t j, int64_t k) {
        return this->data[static_cast<size_t>((i * this->dim(1) + j) * this->dim(2) + k)];
    }
    Real operator()(int64_t i, int64_t j, int64_t k) const {
        return this->data[static_cast<size_t>((i * this->dim(1) + j) * this->dim(2) + k)];
    }
    void fill(Real v) { std::fill(this->data.begin(), this->data.end(), v); }
    void scale_(Real s) {
        for (Real& v : this->data) v *= s;
    }
};

template <class Real>
double l2_norm(const oomb::Tensor<Real>& t) {
    double s = 0.0;
    for (Real v : t.data) s += static_cast<double>(v) * static_cast<double>(v);
    return std::sqrt(s);
}

// ||a - b||_2 / ||b||_2 (||a - b|| when b is zero), accumulated in double.
template <class Real>
double rel_l2_err(const oomb::Tensor<Real>& a, const oomb::Tensor<Real>& b) {
    if (a.shape != b.shape) throw ShapeError("rel_l2_err: shape mismatch");
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) {
        const double d = static_cast<double>(a.data[i]) - static_cast<double>(b.data[i]);
        num += d * d;
        den += static_cast<double>(b.data[i]) * static_cast<double>(b.data[i]);
    }
    return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

template <class Real>
double max_abs_diff(const oomb::Tensor<Real>& a, const oomb::Tensor<Real>& b) {
    if (a.shape != b.shape) throw ShapeError("max_abs_diff: shape mismatch");
    double m = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i)
        m = std::max(m, std::abs(static_cast<double>(a.data[i]) - static_cast<double>(b.data[i])));
    return m;
}

}  // namespace chunktrain
