// idkit_b200_ext.hpp -- C++ entries the drop-in adds to the reference's idkit
// namespace (the shim integration/idkit_b200_shim.cpp defines them).
//
// The reference has no Gaussian-sketch RID; the north-star
// path composes it from generate -> matmul -> qr_column_pivoted ->
// solve_triangular -> select_columns.  This is that path as one call with the
// reference's value semantics (IdResult of id.hpp:17-22, orientation rule of
// id_auto, id.cpp:78-95).
#pragma once

#include <cstddef>
#include <cstdint>

#include "idkit/id.hpp"
#include "idkit/matrix.hpp"

namespace idkit {

/// Gaussian-sketch randomized ID: Y = Omega M with Omega (k + oversampling) x
/// rows(M) drawn on the device (Philox keyed by seed), cols = the first k
/// pivots of qr_column_pivoted(Y, k), Z = [I | R11^-1 R12] P^T, approx =
/// matmul(select_columns(M, cols), Z).  M = a, or a^T when a has more rows than
/// columns (result.transposed, cols index rows of a), as id_auto does.
/// Throws like the reference: std::invalid_argument for k outside
/// [1, min(rows, cols)], SingularMatrixError for a zero R11 diagonal.
IdResult sketch_rid(const Matrix& a, std::size_t k, std::size_t oversampling, std::uint64_t seed);

}  // namespace idkit
