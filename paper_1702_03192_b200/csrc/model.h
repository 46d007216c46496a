// Packed GBDT model for the MTNN selector (host C++).
//
// Layout follows the reference Dispatcher's one-time pack (selector.py:82-123):
// per tree, arrays of a common width = the largest node count; feat = -1 marks a
// leaf; nodes are numbered in pre-order with the root at 0; an empty ensemble is
// one dummy tree holding a single 0.0 leaf.
#pragma once

#include <stdint.h>

#include <vector>

struct mtnn_model {
  int64_t n_trees = 1;  // packed tree count (>= 1)
  int64_t width = 1;
  int64_t n_features = 8;
  double base_score = 0.0;
  double eta = 1.0;
  std::vector<int64_t> feat, left, right;
  std::vector<double> thresh, leaf;
};

namespace mtnn {
// raw = base; for each tree: walk x[f] < t ? left : right; raw += eta * leaf.
// Exactly the reference's float64 arithmetic (compiled with -ffp-contract=off).
double walk_packed(const int64_t* feat, const double* thresh, const int64_t* left,
                   const int64_t* right, const double* leaf, int64_t n_trees, int64_t width,
                   const double* x, double base_score, double eta);
}  // namespace mtnn
