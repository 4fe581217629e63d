// dfs/tensor.hpp — value types of the drop-in dfs:: API (B200 build).
//
// Same declarations and semantics as the reference's dfs/tensor.hpp
// (/root/reference/proj/include/dfs/tensor.hpp:13-84): row-major binary32
// (Matrix) and binary64 (MatrixD) host matrices. Both are one class template
// here; the library moves them to the device per call (see dfs_gpu.h).
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

namespace dfs {

namespace detail {

template <typename T>
class RowMajor {
 public:
  RowMajor() = default;
  RowMajor(int64_t rows, int64_t cols, T fill = T(0)) : rows_(rows), cols_(cols) {
    if (rows < 0 || cols < 0) throw std::invalid_argument(kShapeError);
    data_.assign(static_cast<size_t>(rows * cols), fill);
  }

  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  int64_t size() const { return rows_ * cols_; }
  bool empty() const { return data_.empty(); }

  T& at(int64_t r, int64_t c) { return data_[index(r, c)]; }
  T at(int64_t r, int64_t c) const { return data_[index(r, c)]; }

  std::span<T> row(int64_t r) { return {data_.data() + r * cols_, static_cast<size_t>(cols_)}; }
  std::span<const T> row(int64_t r) const { return {data_.data() + r * cols_, static_cast<size_t>(cols_)}; }

  std::span<T> values() { return data_; }
  std::span<const T> values() const { return data_; }

  bool all_finite() const {
    for (const T v : data_)
      if (!std::isfinite(v)) return false;
    return true;
  }

  friend bool operator==(const RowMajor&, const RowMajor&) = default;

 private:
  static constexpr const char* kShapeError =
      sizeof(T) == sizeof(float) ? "Matrix: negative shape" : "MatrixD: negative shape";
  size_t index(int64_t r, int64_t c) const { return static_cast<size_t>(r * cols_ + c); }

  int64_t rows_ = 0;
  int64_t cols_ = 0;
  std::vector<T> data_;
};

}  // namespace detail

// N x d token matrices and N x N dense attention matrices (binary32).
using Matrix = detail::RowMajor<float>;
// Block score matrices keep binary64 so rankings match the fp64 oracle sums.
using MatrixD = detail::RowMajor<double>;

}  // namespace dfs
