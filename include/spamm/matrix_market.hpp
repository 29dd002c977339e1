#pragma once
//
// spamm-b200 drop-in: MatrixMarket coordinate I/O, the reference's input and
// output format (/root/reference/proj/core/include/spamm/matrix_market.hpp,
// src/matrix_market.cpp:40-117).  Same names, behaviour and exceptions:
//   * only `%%MatrixMarket matrix coordinate real general`, square, 1-based;
//     std::invalid_argument for other banners / rectangular sizes,
//     std::runtime_error for malformed input;
//   * writing lists the stored nonzeros in row-major order, 1-based, with 17
//     significant digits (values re-read bitwise).
// Writing reads the leaves straight from the device (spg_matrix_download).
//
#include <iosfwd>
#include <string>
#include <vector>

#include "spamm/quadtree.hpp"

namespace spamm {

struct CoordinateData {
  int dimension = 0;
  std::vector<CoordinateEntry> entries;
};

CoordinateData read_matrix_market(std::istream& in);
CoordinateData read_matrix_market_file(const std::string& path);

void write_matrix_market(std::ostream& out, const QuadTreeMatrix& x);
void write_matrix_market_file(const std::string& path, const QuadTreeMatrix& x);

}  // namespace spamm
