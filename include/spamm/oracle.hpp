#pragma once
//
// The reference's dense test helpers (/root/reference/proj/core/include/spamm/
// oracle.hpp): declarations only.  They are the reference's test oracle, so the
// product library (libspamm_ec.so) does NOT define them.  Link a build of the
// unmodified reference src/oracle.cpp against these headers (oracle/Makefile
// target `ref` builds oracle/_ref/libspamm_dense_oracle.so -- test
// infrastructure) and hand the functions to the experiment runners with
// spamm::set_experiment_oracle (experiment.hpp).  DecayModelSpec stays here
// because ExperimentConfig carries it.  Gershgorin bounds of a quadtree matrix
// are computed on the device by spamm::gershgorin_bounds (quadtree.hpp).
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
