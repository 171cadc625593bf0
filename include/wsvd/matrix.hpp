// wsvd/matrix.hpp -- the value type of the wsvd::decode drop-in.
//
// The decode operators exchange dense row-major fp64 matrices (reference
// include/wsvd/matrix.hpp:14-61).  This is the subset of that interface the
// decode API and its callers use: shape, element and row access, raw data,
// appending rows, and max_abs_diff / dot for parity checks.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

namespace wsvd {

class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0)
        : r_(rows), c_(cols), v_(rows * cols, fill) {}
    Matrix(std::size_t rows, std::size_t cols, std::vector<double> values);

    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    std::size_t size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }

    double operator()(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }
    double& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
    std::span<const double> row(std::size_t i) const { return {v_.data() + i * c_, c_}; }
    std::span<double> row(std::size_t i) { return {v_.data() + i * c_, c_}; }
    const std::vector<double>& data() const { return v_; }
    std::vector<double>& data() { return v_; }

    /// Appends one row; the first row fixes the width of an empty matrix.
    void append_row(std::span<const double> values);

private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<double> v_;
};

double dot(std::span<const double> a, std::span<const double> b);
double max_abs_diff(const Matrix& a, const Matrix& b);

}  // namespace wsvd
