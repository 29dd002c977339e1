#pragma once
//
// spamm-b200 drop-in: the reference's dense helpers and synthetic-instance
// generator (/root/reference/proj/core/include/spamm/oracle.hpp, src/oracle.cpp),
// which its experiment runner uses for generated inputs, spectral bounds and
// the small-N density-matrix check.  Host code on dense matrices -- never on
// the GPU product path.  generate_decay_matrix reproduces the reference's bits
// for a given seed (mt19937_64 stream, 53-bit mapping, same arithmetic order).
//
#include <cstdint>
#include <utility>
#include <vector>

#include "spamm/dense_matrix.hpp"

namespace spamm::oracle {

DenseMatrix dense_multiply(const DenseMatrix& a, const DenseMatrix& b);
double dense_frobenius(const DenseMatrix& a);

struct EigenDecomposition {
  std::vector<double> eigenvalues;  // ascending
  DenseMatrix eigenvectors;         // eigenvector k in column k
  int sweeps = 0;
};

EigenDecomposition jacobi_eigendecomposition(DenseMatrix a, double threshold = 1e-14,
                                             int max_sweeps = 100);
DenseMatrix density_matrix_oracle(const DenseMatrix& fock, int occupation);

struct DecayModelSpec {
  int dimension = 0;
  double alpha = 0.5;
  double scale = 0.3;
  double spectral_low = 0.0;
  double spectral_high = 2.0;
  std::uint64_t seed = 0;
};

DenseMatrix generate_decay_matrix(const DecayModelSpec& spec);
std::pair<double, double> gershgorin_bounds(const DenseMatrix& a);

}  // namespace spamm::oracle
