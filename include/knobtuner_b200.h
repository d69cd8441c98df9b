/*
 * knobtuner_b200.h — C ABI of the B200 search-step engine (libknobtuner_b200.so).
 *
 * Drop-in boundary for the data-parallel search step of the reference knob
 * tuner (/root/reference/pkg/src/knobtuner).  The reference is pure Python;
 * its "plugin API" is the set of module-level functions the driver imports
 * by name (driver.py:12-23).  Each entry point below replaces one of them (or
 * the array kernel inside one of them) and is bound from Python by
 * paper_1905_12799_b200/_lib.py (ctypes); INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Plain C types only: pointers + sizes.  "_dev" pointers are CUDA device
 *     memory on the engine's device; everything else is host memory.
 *   - A configuration is a "row": one uint64 holding the n_knobs (<= 8) knob
 *     indices.  When every cardinality is <= 255 knob i's index is byte i
 *     (unused high bytes 0); otherwise knob i occupies the bit field
 *     [shift_i, shift_i + width_i) with width_i = max(1, bit_length(card_i - 1))
 *     packed from bit 0 upwards, at most 63 bits in all (cards <= 65535).  Every
 *     entry point that reads rows takes the cardinalities (directly or through
 *     the forest / landscape handle) and derives the same layout.
 *   - Every call returns KT_OK or an error code; kt_last_error() gives the
 *     message.  Error codes map 1:1 onto the reference's exception types so
 *     the Python shim re-raises the same class with the same message
 *     (errors.py:4-41, agent.py:274-277, sampler.py:86-87, cost_model.py:183-184).
 *   - Calls are stream-ordered on the engine's stream; functions that return
 *     host results synchronise that stream before returning.
 */
#ifndef KNOBTUNER_B200_H
#define KNOBTUNER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum {
    KT_OK = 0,
    KT_ERR_VALUE = 1,       /* -> ValueError                                   */
    KT_ERR_DIMENSION = 2,   /* -> knobtuner.errors.DimensionMismatchError       */
    KT_ERR_SPACE = 3,       /* -> knobtuner.errors.SpaceValidationError         */
    KT_ERR_UNSUPPORTED = 4, /* -> NotImplementedError (outside the engine's scope) */
    KT_ERR_CUDA = 10,       /* -> RuntimeError                                  */
    KT_ERR_INTERNAL = 11    /* -> RuntimeError                                  */
};

const char* kt_last_error(void);
const char* kt_version(void);

/* Row layout of a space (host only, no device needed): per-knob bit shift and
 * width, byte-per-knob when every cardinality is <= 255 (see Conventions).   */
int kt_row_layout(const int32_t* cards, int n_knobs, int32_t* shift_out, int32_t* width_out);

/* ------------------------------------------------------------------ engine */
/* One engine per device: owns a CUDA stream and a growable device workspace. */
typedef struct kt_engine kt_engine;

int kt_engine_create(int device, kt_engine** out);
int kt_engine_destroy(kt_engine* e);
/* Use a caller-owned stream (cudaStream_t) instead of the engine's own; NULL restores it. */
int kt_engine_set_stream(kt_engine* e, void* cuda_stream);
int kt_engine_synchronize(kt_engine* e);
/* Order the engine stream and another CUDA stream without a host synchronisation:
 * after = 0: the engine waits for `other`'s work so far; 1: `other` waits for the engine's. */
int kt_engine_order(kt_engine* e, void* other_cuda_stream, int after);
/* Number of engine kernels launched since creation (evidence counter for the bench). */
int64_t kt_engine_launch_count(const kt_engine* e);
/* Per-kernel CUDA-event timing on the engine stream (off by default). */
int kt_engine_set_timing(kt_engine* e, int enabled);
/* Accumulated per-kernel stats: names is capacity x 32 chars; reset != 0 clears them. */
int kt_engine_kernel_stats(kt_engine* e, int capacity, char* names, int64_t* counts, double* total_ms,
                           int32_t* n_kernels, int reset);

/* ------------------------------------------------------- host RNG streams */
/* numpy SeedSequence(entropy, spawn_key) -> PCG64 -> random()/integers(0, n)
 * (numpy/random/bit_generator.pyx SeedSequence, _pcg64.pyx, pcg64.h), used for
 * the seeds the reference derives at sampler.py:89, sa.py:79-81, agent.py:292-296.
 * words = little-endian 32-bit words of the entropy int (at least one word).   */
int kt_pcg64_draw(const uint32_t* entropy_words, int n_entropy_words,
                  const uint32_t* spawn_words, int n_spawn_words,
                  int kind /* 0: random() doubles, 1: integers(0, bound) */,
                  uint64_t bound, int64_t count, void* out /* double[] or int64[] */);

/* --------------------------------------------------- surrogate scoring (K2) */
/* Replaces CostModel._packed + predict_features (cost_model.py:157-201) and
 * predict (cost_model.py:401-409).  The forest is given in the reference's
 * flat per-tree arrays (Tree, cost_model.py:69-77) concatenated; node_offset
 * has n_trees+1 entries.  feature_table is the (n_knobs x max_card) table of
 * log2(1 + knob value) computed by the host exactly as feature_table() does
 * (cost_model.py:235-249); thresholds become per-node index cut points.      */
typedef struct kt_forest kt_forest;

int kt_forest_create(kt_engine* e, int n_knobs, const int32_t* cards,
                     const double* feature_table, int max_card,
                     int n_trees, const int32_t* node_offset,
                     const int32_t* feature, const double* threshold,
                     const int32_t* child_left, const int32_t* child_right,
                     const double* value, double base_score, kt_forest** out);
int kt_forest_destroy(kt_forest* f);
int kt_forest_depth(const kt_forest* f);
/* scores_dev[i] = surrogate fitness of rows_dev[i] (bit-exact with predict_features). */
int kt_score_trees(kt_engine* e, const kt_forest* f, const uint64_t* rows_dev,
                   int64_t count, double* scores_dev);

/* ------------------------------------------------ landscape scoring (K3) */
/* Replaces synthetic_runtime/_hash_unit (backends.py:157-174) and
 * SyntheticBackend.batch_runtimes (backends.py:272-273), bit-exact (glibc's exp restated
 * on the device).  seed_text is str(landscape.seed) (the blake2b payload prefix).                        */
typedef struct kt_landscape kt_landscape;

int kt_landscape_create(kt_engine* e, int n_knobs, const int32_t* cards, int n_centers, const int32_t* centers,
                        const double* depths, const double* radii, double base_runtime,
                        double noise_rel, const char* seed_text, kt_landscape** out);
int kt_landscape_destroy(kt_landscape* l);
int kt_score_landscape(kt_engine* e, const kt_landscape* l, const uint64_t* rows_dev,
                       int64_t count, double* runtime_dev);
/* Brute-force optimum over the whole lattice (cli.py:77-90 _enumerated_oracle, without the
 * enumerate_space cap of space.py:20): *best_runtime = the minimum runtime, *best_rank = its
 * lexicographic rank in enumerate_space order (last knob fastest), the first one on ties. */
int kt_landscape_best(kt_engine* e, const kt_landscape* l, const int32_t* cards,
                      double* best_runtime, int64_t* best_rank);

/* ---------------------------------------------------- adaptive sampling */
/* First-occurrence dedup (sampler.py:187-192): distinct_dev receives the
 * distinct rows in order of first occurrence; *n_distinct their count.     */
int kt_dedup(kt_engine* e, const uint64_t* rows_dev, int64_t count,
             uint64_t* distinct_dev, int64_t* n_distinct);

/* Per-knob mode over all rows, ties -> smallest index (mode_config, sampler.py:151-158). */
int kt_mode_vote(kt_engine* e, const uint64_t* rows_dev, int64_t count,
                 int n_knobs, const int32_t* cards, int32_t* mode_out);

/* Seeded k-means on lattice points (kmeans, sampler.py:72-122).
 * assignment_out: host int64[m] (may be NULL); centroids_out: host double[k*n];
 * history_out: host double[100] (may be NULL: then only the final loss is
 * computed); returns the number of Lloyd passes in *n_passes.               */
int kt_kmeans(kt_engine* e, const uint64_t* points_dev, int64_t m, int n_knobs,
              const int32_t* cards, int k, uint64_t seed, double* centroids_out, int64_t* assignment_out,
              double* loss_out, double* history_out, int32_t* n_passes);

/* Knee scan (knee_scan, sampler.py:125-148): grows k from 8 until
 * knee_constant * L_k > L_{k-1}; returns the breaking k's clustering.
 * scanned_k/scanned_loss: host arrays of capacity 56.                       */
int kt_knee_scan(kt_engine* e, const uint64_t* points_dev, int64_t m, int n_knobs,
                 const int32_t* cards, uint64_t seed, double knee_constant, int k_max,
                 int32_t* scanned_k, double* scanned_loss, int32_t* n_scanned,
                 double* centroids_out /* k_max*n */, int64_t* assignment_out /* m or NULL */);

/* Statistics of one adaptive_sample call. */
typedef struct kt_sample_info {
    int64_t n_distinct;     /* m */
    int32_t chosen_k;       /* 0 when the <=8-distinct bypass was taken */
    int32_t n_scanned;
    int32_t scanned_k[56];
    double scanned_loss[56];
    int32_t lloyd_passes;   /* sum over scanned k */
    int32_t used_mode;      /* 1 if a visited centroid was replaced by the mode */
    int32_t lloyd_launches; /* fused multi-k Lloyd launches */
    int64_t lloyd_bytes;    /* algorithmic bytes of all Lloyd passes: per pass m*n point
                               bytes + 2*m assignment bytes per active k */
} kt_sample_info;

/* The whole adaptive_sample (sampler.py:173-215): dedup -> knee k-means ->
 * round centroids -> visited/mode replacement -> dedup of the batch.
 * visited_rows: host array of measured configurations (VisitedSet).
 * batch_out: host, capacity 63 rows.                                        */
/* _top_unvisited (driver.py:101-115), the non-adaptive arms' batch: the first occurrence of every
 * trajectory row not in visited[0, n_visited) (host array, any order), stable-sorted by descending
 * score; the first `cap` (<= 64) rows -> batch_out (host), their count -> *batch_len.              */
int kt_top_unvisited(kt_engine* e, const uint64_t* rows_dev, const double* scores_dev, int64_t count,
                     const uint64_t* visited, int64_t n_visited, int cap, uint64_t* batch_out, int32_t* batch_len);

int kt_adaptive_sample(kt_engine* e, const uint64_t* rows_dev, int64_t count,
                       int n_knobs, const int32_t* cards,
                       const uint64_t* visited_rows, int64_t n_visited,
                       uint64_t seed, double knee_constant,
                       uint64_t* batch_out, int32_t* batch_len, kt_sample_info* info);

/* ------------------------------------------------ simulated annealing (K10) */
/* run_sa_round (sa.py:62-122).  The first min(n_starts, chains) rows of
 * starts_dev are used; missing starts are padded from the parent stream
 * exactly like sa.py:83-85.  Chain c's PCG64 stream is derived on the device
 * from SeedSequence(seed, spawn_key=(c,)) (sa.py:79-81).  Outputs are the
 * reference's chain-major trajectory (start, then each accepted move), compact:
 * rows/scores/step indices, *n_out entries; capacity chains * (steps + 1).
 * seed_words: little-endian 32-bit words of seed & (2^64 - 1).            */
int kt_sa_chains(kt_engine* e, const kt_forest* f, const uint64_t* starts_dev, int32_t n_starts,
                 int32_t chains, int32_t steps, const int32_t* cards, int n_knobs,
                 const uint32_t* seed_words, int n_seed_words,
                 int has_initial_temperature, double initial_temperature, double cooling,
                 uint64_t* rows_out_dev, double* scores_out_dev, int32_t* steps_out_dev,
                 int64_t* n_out);

/* -------------------------------------------- PPO search agents (K1, K4, K5) */
/* Device-resident actor-critic (nets.py:8-10 layout, PARAM_KEYS order) with
 * float64 master weights and Adam moments (Agent, agent.py:130-176).        */
typedef struct kt_agent kt_agent;

typedef struct kt_ppo_hyper {
    double adam_step_size, discount, gae_parameter, clip, value_coef, entropy_coef;
    int32_t epochs, max_steps;
} kt_ppo_hyper;

typedef struct kt_round_info {
    int64_t steps;    /* T: PPO rows (agent steps) */
    int64_t entries;  /* N = T + episodes: trajectory entries */
    int64_t guarded;  /* reserved: 0 (the float64 rollout re-decides nothing) */
    double policy_loss, value_loss, entropy, total;  /* final-epoch LossReport */
    double guard_tau; /* reserved: 0 */
} kt_round_info;

int kt_agent_create(kt_engine* e, int n_knobs, int shared_width, int head_width, const double* params,
                    const double* adam_m, const double* adam_v, int64_t adam_t, kt_agent** out);
int kt_agent_destroy(kt_agent* a);
/* Copy the device state back (params / Adam moments in PARAM_KEYS order). */
int kt_agent_get_state(kt_engine* e, const kt_agent* a, double* params, double* adam_m, double* adam_v,
                       int64_t* adam_t);
/* One search round (run_search_round, agent.py:267-366) for max_steps >= 1:
 * rollout of E episodes (episode e's uniforms from
 * SeedSequence(seed, spawn_key=(round_index, e))), surrogate scores of every
 * visited configuration, reward / GAE / advantage normalisation and `epochs`
 * PPO+Adam updates.  Outputs the episode-major trajectory: rows, scores and
 * step indices (capacity E * (max_steps + 1)), *n_out entries.            */
int kt_search_round(kt_engine* e, kt_agent* a, const kt_forest* f, const uint64_t* starts_dev, int32_t E,
                    const int32_t* cards, int n_knobs, const uint32_t* seed_words, int n_seed_words,
                    int64_t round_index, const kt_ppo_hyper* hyper, uint64_t* rows_out_dev,
                    double* scores_out_dev, int32_t* steps_out_dev, int64_t* n_out, kt_round_info* info,
                    double* logp_out_dev /* T or NULL */, double* values_out_dev /* T or NULL */);

/* ------------------------------------------------ sharded k-means (multi-GPU)
 * One rank's contiguous, pairwise-tree-aligned shard of the distinct points
 * (SURVEY §8(e)); replaces the Lloyd loop of kmeans (sampler.py:91-116) for that
 * shard.  Per pass the host calls kt_lloyd_pass (fills ext_dev, int64
 * [K*9 + R]: per-cluster coordinate/count deltas, then per-run changed counts),
 * all-reduces ext_dev with SUM over the ranks (NCCL), then kt_lloyd_apply (sums
 * += deltas; converged / maxed / reseed / active per run, identical on every
 * rank).  init_rows: host, max(ks) k-means++ rows (kt_kmeanspp_rows).         */
typedef struct kt_lloyd kt_lloyd;
int kt_lloyd_create(kt_engine* e, const uint64_t* shard_pts_dev, int64_t shard_m, int n_knobs, const int32_t* cards,
                    int n_runs, const int32_t* ks, const uint64_t* init_rows, kt_lloyd** out);
int kt_lloyd_destroy(kt_lloyd* l);
int kt_lloyd_clusters(const kt_lloyd* l, int32_t* n_clusters);
int kt_lloyd_pass(kt_engine* e, kt_lloyd* l, uint64_t* ext_dev);
/* states_out[r]: 0/1/5 active, 2 converged, 3 maxed (100 passes), 4 needs reseed. */
int kt_lloyd_apply(kt_engine* e, kt_lloyd* l, const uint64_t* ext_dev, int32_t* states_out, int32_t* passes_out);
/* Native NCCL communicator (loaded with dlopen; the unique id travels over the caller's
 * process group) for the two exchanges north_star names, both on the engine stream with no
 * host round trip: the k-means partial sums (sampler.py:94-115) and the PPO gradient /
 * round-statistics all-reduce (agent.py:245-257).  kt_comm_all_reduce_f64 has the
 * kt_all_reduce_f64_fn signature: pass it with user = the kt_comm* in a kt_collective.      */
typedef struct kt_comm kt_comm;
int kt_comm_unique_id(uint8_t* id_out /* 128 bytes */);
int kt_comm_create(kt_engine* e, const uint8_t* id, int rank, int world, kt_comm** out);
int kt_comm_destroy(kt_comm* c);
int kt_comm_all_reduce_f64(void* comm, double* dev_buf, int64_t count);
int kt_comm_all_reduce_i64(kt_comm* c, int64_t* dev_buf, int64_t count);
/* Device-driven sharded Lloyd loop: enqueues `batch` rounds of pass -> ncclAllReduce(int64,
 * comm; NULL = one rank) -> apply per host check (the iteration counter lives on the device);
 * returns when no run is active or a run needs a reseed (*reseed_out = 1: do the host reseed
 * with kt_lloyd_sums / kt_lloyd_farthest / kt_lloyd_set_centroids, then call again).
 * Replaces the per-pass kt_lloyd_pass / all-reduce / kt_lloyd_apply host loop. */
int kt_lloyd_run(kt_engine* e, kt_lloyd* l, kt_comm* comm, int batch, int32_t* states_out, int32_t* passes_out,
                 int32_t* reseed_out);
/* Global cluster sums (host int64 [K][9]: 8 coordinate sums, count). */
int kt_lloyd_sums(kt_engine* e, kt_lloyd* l, int64_t* sums_out);
/* Empty-cluster reseed (sampler.py:108-115): the shard's farthest point from its
 * assigned centroid under the last pass, skipping `blocked` (shard-local indices);
 * *idx_out = -1 when none is left.                                          */
int kt_lloyd_farthest(kt_engine* e, kt_lloyd* l, int run, const int64_t* blocked, int n_blocked, double* d2_out,
                      int64_t* idx_out);
/* Centroids for the next pass of `run` (host double [k*n]), e.g. after a reseed. */
int kt_lloyd_set_centroids(kt_engine* e, kt_lloyd* l, int run, const double* centroids);
/* Centroids the last pass of `run` used (host double [k*n]). */
int kt_lloyd_centroids(kt_engine* e, kt_lloyd* l, int run, double* centroids_out);
int kt_lloyd_assignment(kt_engine* e, kt_lloyd* l, int run, int64_t* assignment_out /* shard_m */);
/* numpy pairwise loss of each leaf [bounds[i], bounds[i+1]) of the shard (host double [n_leaves]). */
int kt_lloyd_leaf_losses(kt_engine* e, kt_lloyd* l, int run, const int64_t* bounds, int n_leaves, double* out);
/* k-means++ rows (_plus_plus_init, sampler.py:56-69) of k centroids; host uint64 [k]. */
int kt_kmeanspp_rows(kt_engine* e, const uint64_t* points_dev, int64_t m, int n_knobs, const int32_t* cards,
                     uint64_t seed, int k, uint64_t* rows_out);

/* Sharded search round: this rank's episodes are the global
 * episodes [episode_offset, episode_offset + E) — their uniforms come from
 * SeedSequence(seed, spawn_key=(round_index, episode_offset + e)) — and the
 * reward / advantage statistics, the PPO batch size, the per-epoch gradients
 * (float64, PARAM_KEYS order) and the loss report are summed over the ranks
 * through all_reduce_sum_f64: an in-place SUM of `count` device doubles,
 * ordered on the engine stream (NCCL under torch.distributed in the Python
 * layer), returning 0 on success.  Every rank then applies the same Adam step.
 * Replaces run_search_round (agent.py:267-366) for one shard of the agents.  */
typedef int (*kt_all_reduce_f64_fn)(void* user, double* dev_buf, int64_t count);
typedef struct kt_collective {
    kt_all_reduce_f64_fn all_reduce_sum_f64;
    void* user;
    int64_t episode_offset;
} kt_collective;
int kt_search_round_ex(kt_engine* e, kt_agent* a, const kt_forest* f, const uint64_t* starts_dev, int32_t E,
                       const int32_t* cards, int n_knobs, const uint32_t* seed_words, int n_seed_words,
                       int64_t round_index, const kt_ppo_hyper* hyper, uint64_t* rows_out_dev,
                       double* scores_out_dev, int32_t* steps_out_dev, int64_t* n_out, kt_round_info* info,
                       double* logp_out_dev, double* values_out_dev, const kt_collective* coll /* NULL: 1 rank */);

/* compute_gae (agent.py:191-210) of E episodes laid out episode-major: rewards / values [T]
 * float64 (device), lengths [E] int32 (device), terminal value 0; adv_out [T] (device).
 * The same kernel the PPO update runs (float64, the reference's reverse recurrence). */
int kt_gae(kt_engine* e, const double* rewards_dev, const double* values_dev, const int32_t* lengths_dev, int32_t E,
           double discount, double gae_parameter, double* adv_out_dev);

/* ------------------------------------------------ surrogate refit
 * Gradient-boosted regression trees, exact greedy squared error (fit,
 * cost_model.py:367-398; _grow :328-364; _best_split :292-325), host code in
 * numpy's operation order: byte-identical models.  features: host double
 * [m][n] row-major; outputs: every tree's nodes in preorder (feature -1 =
 * leaf), concatenated; tree_offsets_out[r] = first node of tree r (rounds + 1
 * entries); node_capacity >= rounds * (2^(depth+1) - 1).  No device work.   */
int kt_fit_trees(const double* features, const double* targets, int64_t m, int n, int rounds, int depth,
                 double learning_rate, int32_t* feature_out, double* threshold_out, int32_t* left_out,
                 int32_t* right_out, double* value_out, int64_t node_capacity, int32_t* tree_offsets_out,
                 double* base_out);

/* Same contract and bytes as kt_fit_trees, with the boosting loop on the GPU: one single-CTA
 * kernel grows every tree (a warp per node of a level, a lane per feature for the split scans,
 * float64 in the reference's operation order); the host only sorts (canonical lexsort order,
 * per-feature stable argsorts).  depth <= 7, n_features <= 8 (else KT_ERR_UNSUPPORTED).
 * Replaces cost_model.py:367-398 (fit) on the device path of the tuning loop (driver.py:142-148). */
int kt_fit_trees_device(kt_engine* engine, const double* features, const double* targets, int64_t m, int n,
                        int rounds, int depth, double learning_rate, int32_t* feature_out, double* threshold_out,
                        int32_t* left_out, int32_t* right_out, double* value_out, int64_t node_capacity,
                        int32_t* tree_offsets_out, double* base_out);

/* ------------------------------------------------ trajectory analysis
 * per_step_best (report.py:53-69): best_out[s] = max score of the entries landing at step s
 * (-inf if none), s < cap; *horizon_out = max step index.  pca_project (report.py:227-253):
 * exact int64 moments sums_out[n] = sum x_i, gram_out[n*n] = sum x_i x_j, then projections
 * xs/ys (device doubles) = (x - mean) . v1 / v2.                                         */
int kt_step_best(kt_engine* e, const double* scores_dev, const int32_t* steps_dev, int64_t count, int cap,
                 double* best_out, int32_t* horizon_out);
int kt_pca_moments(kt_engine* e, const uint64_t* rows_dev, int64_t count, int n_knobs, const int32_t* cards,
                   int64_t* sums_out, int64_t* gram_out);
int kt_pca_project(kt_engine* e, const uint64_t* rows_dev, int64_t count, int n_knobs, const int32_t* cards,
                   const double* mean, const double* v1, const double* v2, double* xs_dev, double* ys_dev);

/* ------------------------------------------------------------ utilities */
/* fp32 GEMM on the tensor cores (tcgen05 kind::tf32, 3xTF32 split, fp32 accumulate
 * in TMEM): C[m][n] = sum_k A(m,k) B(k,n), row-major device arrays;
 * A(m,k) = trans_a ? A[k*lda+m] : A[m*lda+k], B(k,n) = trans_b ? B[n*ldb+k] : B[k*ldb+n].
 * Used by the PPO update; exported for verification.                        */
int kt_gemm_f32(kt_engine* e, int trans_a, int trans_b, int M, int N, int K, const float* A, int lda,
                const float* B, int ldb, float* C, int ldc);

#ifdef __cplusplus
}
#endif

#endif /* KNOBTUNER_B200_H */
