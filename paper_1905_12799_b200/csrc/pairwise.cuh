// pairwise.cuh — numpy's pairwise summation order on the device.
//
// numpy reduces a contiguous float64 array with pairwise_sum
// (numpy/_core/src/umath/loops_utils.h.src): blocks of <= 128 values summed
// with 8 strided accumulators, larger ranges split at n2 = n/2 - (n/2 % 8).
// The split tree depends only on the length, so it is built once per length
// on the host; leaves are summed one per thread and the tree is combined
// level by level in a single block.  Used for the k-means loss
// (sampler.py:97-98) and numpy mean/std (sa.py:93-97, agent.py:344-349).
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace kt {

struct PairwiseTree {
    int64_t m = 0;
    std::vector<int64_t> leaf_start;
    std::vector<int32_t> leaf_len;
    std::vector<int32_t> node_left, node_right;  // internal nodes, ids >= L
    std::vector<int32_t> level_start;            // internal nodes grouped by height
    int64_t* d_leaf_start = nullptr;
    int32_t* d_leaf_len = nullptr;
    int32_t* d_left = nullptr;
    int32_t* d_right = nullptr;
    int32_t* d_level = nullptr;
    int root = 0;
    int n_levels = 0;
    void* d_block = nullptr;  // the five device arrays above, one allocation
    ~PairwiseTree() { cudaFree(d_block); }
};

std::shared_ptr<const PairwiseTree> pairwise_tree(int device, int64_t m);

// k-means loss: sum over points of the float64 squared distance to the assigned centroid.
void pairwise_loss(kt_engine* e, const uint64_t* pts, int64_t m, int n, const RowFmt& fmt, const uint8_t* assign,
                   const double* cent,
                   double* out_dev);

// The losses of R <= kMaxLossRuns runs over the same points in two launches: run r's
// assignment is assign + r * astride, its centroids cent + coff[r] * kMaxKnobs.
constexpr int kMaxLossRuns = 8;
void pairwise_loss_runs(kt_engine* e, const uint64_t* pts, int64_t m, int n, const RowFmt& fmt, const uint8_t* assign,
                        int64_t astride, const double* cent, const int* coff, int R, double* out_dev);

// numpy sum of x[0..m) (center == nullptr) or of (x - *center)^2 (center: device scalar).
void pairwise_sum(kt_engine* e, const double* x, int64_t m, const double* center, double* out_dev);

}  // namespace kt
