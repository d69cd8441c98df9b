// trees.cu — K2 score_trees: boosted-tree surrogate over packed lattice rows.
//
// Replaces CostModel._packed / predict_features (cost_model.py:157-201) and the
// featurize step in front of it (cost_model.py:252-261).
//
// Host packing (kt_forest_create):
//   * every tree is re-laid as a complete binary heap of the forest's maximum
//     depth D; a leaf above depth D becomes an "always left" split whose two
//     children both carry the leaf value, so the walk is a fixed D steps;
//   * a float threshold on feature f = log2(1 + value) is converted to an index
//     cut point t = #{v : table[f][v] <= threshold}; since the table is
//     non-decreasing in the index, "x[f] <= threshold" <=> "idx[f] < t", so the
//     device never touches floating-point features (exactly the reference's
//     routing, cost_model.py:197-198);
//   * node entries are 16 bit (feature << 12 | cut: one PRMT with the entry as its
//     selector puts the knob's byte on top, one compare against cut << 24); a node and its two children
//     are packed into one 64-bit "super node", so one shared-memory load
//     resolves two levels (3 LDS per depth-4 tree instead of 5).
//
// Device walk: leaf values are accumulated in float64 in tree order and the
// base score is added last — numpy's axis-0 sum of the (trees, rows) leaf
// matrix is sequential, so this is bit-exact with the reference.
#include <algorithm>
#include <cstring>
#include <cmath>
#include <vector>

#include "forest.cuh"

namespace kt {

static int super_words(int D) {
    int w = 0;
    for (int d = 0; d < D; d += 2) w += 1 << d;
    return w;
}

static int tree_depth(const int32_t* feat, const int32_t* left, const int32_t* right, int node, int count, int guard) {
    if (node < 0 || node >= count) fail(KT_ERR_VALUE, "tree child index out of range");
    if (guard > 64) fail(KT_ERR_VALUE, "tree deeper than 64 levels (cycle?)");
    if (feat[node] < 0) return 0;
    int a = tree_depth(feat, left, right, left[node], count, guard + 1);
    int b = tree_depth(feat, left, right, right[node], count, guard + 1);
    return 1 + std::max(a, b);
}

namespace {
struct Packer {
    int D, n;
    const int32_t* cards;
    const double* table;
    int max_card;
    bool wide;
    const int32_t *feat, *left, *right;
    const double *thr, *val;
    std::vector<uint16_t> heap;  // 2^D - 1 internal entries
    std::vector<double> leaf;    // 2^D leaves

    uint16_t entry_for(int node) const {
        int f = feat[node];
        if (f >= n) fail(KT_ERR_DIMENSION, "tree splits on feature " + std::to_string(f) + " but the space has " +
                                               std::to_string(n) + " knobs");
        int card = cards[f];
        const double* row = table + size_t(f) * max_card;
        int cut = 0;
        while (cut < card && row[cut] <= thr[node]) ++cut;  // table is non-decreasing
        return uint16_t(wide ? (f | (cut << 3)) : ((f << 12) | cut));
    }
    void fill(int node, int h, int depth) {
        if (depth == D) {
            leaf[h - ((1 << D) - 1)] = val[node];  // node is a leaf here by construction
            return;
        }
        if (feat[node] < 0) {
            heap[h] = uint16_t(wide ? (8191 << 3) : 255);  // idx < cut always: left
            fill(node, 2 * h + 1, depth + 1);
            fill(node, 2 * h + 2, depth + 1);
        } else {
            heap[h] = entry_for(node);
            fill(left[node], 2 * h + 1, depth + 1);
            fill(right[node], 2 * h + 2, depth + 1);
        }
    }
};
}  // namespace

// Rows are processed two per thread for memory/LDS latency overlap.
template <int D, bool WIDE>
__global__ void __launch_bounds__(256) score_trees_kernel(const uint64_t* __restrict__ forest, int words_per_tree,
                                                          int t0, int t1, int n_trees, double base,
                                                          const uint64_t* __restrict__ rows, int64_t count,
                                                          double* __restrict__ out, const RowFmt fmt) {
    extern __shared__ uint64_t s_forest[];
    const int nt = t1 - t0;
    const int total = nt * words_per_tree;
    const uint64_t* src = forest + size_t(t0) * words_per_tree;
    for (int i = threadIdx.x; i < total; i += blockDim.x) s_forest[i] = src[i];
    __syncthreads();

    const bool first_chunk = t0 == 0, last_chunk = t1 == n_trees;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 2;
    for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < count; i += stride) {
        const bool two = i + 1 < count;
        uint64_t r0 = rows[i];
        uint64_t r1 = two ? rows[i + 1] : r0;
        uint32_t lo0 = uint32_t(r0), hi0 = uint32_t(r0 >> 32);
        uint32_t lo1 = uint32_t(r1), hi1 = uint32_t(r1 >> 32);
        WideRow x0{}, x1{};
        if constexpr (WIDE) {
            x0 = widen_row(r0, fmt);
            x1 = widen_row(r1, fmt);
        }
        auto walk = [&](const uint64_t* tr, int which) -> double {
            if constexpr (WIDE) return walk_tree_wide<D>(tr, which ? x1 : x0);
            else return walk_tree<D>(tr, which ? lo1 : lo0, which ? hi1 : hi0);
        };
        double a0, a1;
        int t = 0;
        if (first_chunk) {
            a0 = walk(s_forest, 0);
            a1 = walk(s_forest, 1);
            t = 1;
        } else {
            a0 = out[i];
            a1 = two ? out[i + 1] : 0.0;
        }
#pragma unroll 2
        for (; t < nt; ++t) {
            const uint64_t* tr = s_forest + t * words_per_tree;
            a0 = __dadd_rn(a0, walk(tr, 0));
            a1 = __dadd_rn(a1, walk(tr, 1));
        }
        if (last_chunk) {
            a0 = __dadd_rn(base, a0);
            a1 = __dadd_rn(base, a1);
        }
        out[i] = a0;
        if (two) out[i + 1] = a1;
    }
}

__global__ void fill_kernel(double* out, int64_t count, double v) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = v;
}

template <int D, bool WIDE>
static void launch_score_t(kt_engine* e, const kt_forest* f, const uint64_t* rows, int64_t count, double* out) {
    const int threads = 256;
    const size_t bytes_per_tree = size_t(f->words_per_tree) * 8;
    const size_t smem_cap = 96 * 1024;
    int per_chunk = int(std::max<size_t>(1, smem_cap / bytes_per_tree));
    per_chunk = std::min(per_chunk, f->n_trees);
    const size_t smem = size_t(per_chunk) * bytes_per_tree;
    auto kern = score_trees_kernel<D, WIDE>;
    allow_dynamic_smem((const void*)kern);
    int occ = occupancy_blocks((const void*)kern, threads, smem);
    int64_t want = ceil_div(count, threads * 2);
    int grid = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(e->num_sms) * std::max(occ, 1))));
    for (int t0 = 0; t0 < f->n_trees; t0 += per_chunk) {
        int t1 = std::min(f->n_trees, t0 + per_chunk);
        e->pre_launch("score_trees");
        kern<<<grid, threads, size_t(t1 - t0) * bytes_per_tree, e->stream>>>(
            f->dev, f->words_per_tree, t0, t1, f->n_trees, f->base, rows, count, out, f->fmt);
        e->check_launch("score_trees");
    }
}

template <int D>
static void launch_score(kt_engine* e, const kt_forest* f, const uint64_t* rows, int64_t count, double* out) {
    if (f->wide) launch_score_t<D, true>(e, f, rows, count, out);
    else launch_score_t<D, false>(e, f, rows, count, out);
}

void score_trees(kt_engine* e, const kt_forest* f, const uint64_t* rows, int64_t count, double* out) {
    if (count <= 0) return;
    if (f->n_trees == 0) {
        int grid = int(std::min<int64_t>(ceil_div(count, 256), int64_t(e->num_sms) * 8));
        e->pre_launch("fill");
        fill_kernel<<<grid, 256, 0, e->stream>>>(out, count, f->base);
        e->check_launch("fill");
        return;
    }
    switch (f->depth) {
        case 1: launch_score<1>(e, f, rows, count, out); break;
        case 2: launch_score<2>(e, f, rows, count, out); break;
        case 3: launch_score<3>(e, f, rows, count, out); break;
        case 4: launch_score<4>(e, f, rows, count, out); break;
        case 5: launch_score<5>(e, f, rows, count, out); break;
        case 6: launch_score<6>(e, f, rows, count, out); break;
        case 7: launch_score<7>(e, f, rows, count, out); break;
        case 8: launch_score<8>(e, f, rows, count, out); break;
        default: fail(KT_ERR_UNSUPPORTED, "tree depth > 8 is not supported by the engine");
    }
}

}  // namespace kt

extern "C" {

int kt_forest_create(kt_engine* e, int n_knobs, const int32_t* cards, const double* feature_table, int max_card,
                     int n_trees, const int32_t* node_offset, const int32_t* feature, const double* threshold,
                     const int32_t* child_left, const int32_t* child_right, const double* value, double base_score,
                     kt_forest** out) {
    KT_API_BEGIN
    using namespace kt;
    if (n_knobs < 1 || n_knobs > kMaxKnobs)
        fail(KT_ERR_UNSUPPORTED, "engine rows hold 1..8 knobs, got " + std::to_string(n_knobs));
    const RowFmt fmt = row_fmt(cards, n_knobs);
    for (int i = 0; i < n_knobs; ++i) {
        if (cards[i] > max_card) fail(KT_ERR_VALUE, "feature table narrower than a knob's cardinality");
        if (!fmt.bytes && cards[i] > 8191) fail(KT_ERR_UNSUPPORTED, "tree cut points support at most 8191 settings");
    }
    auto* f = new kt_forest();
    f->fmt = fmt;
    f->wide = !fmt.bytes;
    f->n_knobs = n_knobs;
    f->n_trees = n_trees;
    f->base = base_score;
    f->device = e->device;
    int D = 1;
    for (int t = 0; t < n_trees; ++t) {
        int lo = node_offset[t], hi = node_offset[t + 1];
        if (hi <= lo) fail(KT_ERR_VALUE, "empty tree");
        D = std::max(D, tree_depth(feature + lo, child_left + lo, child_right + lo, 0, hi - lo, 0));
    }
    if (D > 8) fail(KT_ERR_UNSUPPORTED, "tree depth > 8 is not supported by the engine");
    f->depth = D;
    const int sw = super_words(D);
    f->words_per_tree = sw + (1 << D);
    f->host.assign(size_t(n_trees) * f->words_per_tree, 0);
    for (int t = 0; t < n_trees; ++t) {
        int lo = node_offset[t];
        Packer p{D, n_knobs, cards, feature_table, max_card, !fmt.bytes, feature + lo, child_left + lo, child_right + lo,
                 threshold + lo, value + lo, std::vector<uint16_t>((1 << D) - 1, 0), std::vector<double>(1 << D, 0.0)};
        p.fill(0, 0, 0);
        uint64_t* dst = f->host.data() + size_t(t) * f->words_per_tree;
        int off = 0;
        for (int d = 0; d < D; d += 2) {
            for (int j = 0; j < (1 << d); ++j) {
                int h = (1 << d) - 1 + j;
                uint64_t w = p.heap[h];
                if (d + 1 < D) {
                    w |= uint64_t(p.heap[2 * h + 1]) << 16;
                    w |= uint64_t(p.heap[2 * h + 2]) << 32;
                }
                dst[off + j] = w;
            }
            off += 1 << d;
        }
        for (int j = 0; j < (1 << D); ++j) {
            uint64_t bits;
            std::memcpy(&bits, &p.leaf[j], 8);
            dst[off + j] = bits;
        }
    }
    if (!f->host.empty()) {
        KT_CUDA(cudaSetDevice(e->device));
        KT_CUDA(cudaMalloc(&f->dev, f->host.size() * 8));
        KT_CUDA(cudaMemcpy(f->dev, f->host.data(), f->host.size() * 8, cudaMemcpyHostToDevice));
    }
    *out = f;
    KT_API_END
}

int kt_forest_destroy(kt_forest* f) {
    KT_API_BEGIN
    if (!f) return KT_OK;
    if (f->dev) cudaFree(f->dev);
    delete f;
    KT_API_END
}

int kt_forest_depth(const kt_forest* f) { return f ? f->depth : -1; }

int kt_score_trees(kt_engine* e, const kt_forest* f, const uint64_t* rows_dev, int64_t count, double* scores_dev) {
    KT_API_BEGIN
    kt::score_trees(e, f, rows_dev, count, scores_dev);
    KT_API_END
}

}  // extern "C"
