// quake/buffer.hpp (drop-in) — buffer and matrix-view types.
//
// Source-compatible with the reference's core/include/quake/buffer.hpp
// (:25-38): contiguous fp32 buffers and row-major matrix views with no
// strides — also the layout the GPU kernels read in HBM.
#ifndef QUAKE_B200_QUAKE_BUFFER_HPP_
#define QUAKE_B200_QUAKE_BUFFER_HPP_

#include <cstddef>
#include <span>
#include <vector>

namespace quake {

using NumericBuffer = std::vector<float>;

// Row-major view over a buffer (rows of `cols` consecutive floats).
struct MatrixView {
  std::span<const float> data;
  std::size_t cols;

  std::size_t rows() const { return cols == 0 ? 0 : data.size() / cols; }
  bool well_formed() const { return cols != 0 && data.size() % cols == 0; }
  std::span<const float> row(std::size_t r) const { return data.subspan(r * cols, cols); }
};

}  // namespace quake

#endif  // QUAKE_B200_QUAKE_BUFFER_HPP_
