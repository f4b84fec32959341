/*
 * hanf.h -- C-ABI of the B200 HyperANF engine (libhanf.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The
 * reference (/root/reference/proj/include/hyperanf/) is a header-only C++20
 * library with no FFI; its engine surface is the C++ API in engine.hpp.
 * Each entry point below names the reference interface it replaces.  The
 * C++ wrapper include/hyperanf_b200/engine.hpp restores that exact surface
 * (class names, argument meaning, exception types) on top of this ABI, and
 * paper_1011_5599_b200/ mirrors it for Python.
 *
 * Conventions:
 *  - plain pointers and sizes only; no exceptions cross the ABI;
 *  - every call returns a hanf_status; hanf_last_error() gives the
 *    thread-local message of the last failure;
 *  - graph arrays are caller-owned and copied to HBM at create time;
 *    device buffers are engine-owned;
 *  - a handle is driven by one host thread.
 */
#ifndef HANF_H
#define HANF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hanf_status;
#define HANF_OK 0
#define HANF_INVALID_ARGUMENT 1 /* std::invalid_argument: engine.hpp:71-74, hll.hpp:45-48 */
#define HANF_GUARD 2            /* hyperanf::GuardError: engine.hpp:255-258 */
#define HANF_OUT_OF_RANGE 3     /* std::out_of_range: hll.hpp:233-235 */
#define HANF_CUDA_ERROR 4       /* std::runtime_error (device failure) */
#define HANF_OUT_OF_MEMORY 5    /* std::bad_alloc / cudaErrorMemoryAllocation */
#define HANF_CAPACITY 6         /* caller-provided output buffer too small */
#define HANF_IO_ERROR 7         /* hyperanf::IoError: errors.hpp:13-15 */
#define HANF_PARSE_ERROR 8      /* hyperanf::ParseError: errors.hpp:8-10 */

typedef struct hanf_engine hanf_engine;
typedef struct hanf_graph hanf_graph;

/* Read-only CSR view; replaces `const Graph&` (graph.hpp:23-69): num_nodes
 * (:46), num_arcs (:47), offsets() u64[n+1] (:56), arcs() u32[a] (:57).
 * Successor lists need not be sorted or deduplicated for the engine (a
 * union is order- and duplicate-insensitive), but Graph always is. */
typedef struct {
  uint64_t n;
  uint64_t num_arcs;
  const uint64_t* offsets;
  const uint32_t* arcs;
} hanf_graph_view;

/* EngineConfig (engine.hpp:32-46) plus B200 options.  No option changes a
 * single result bit except the sketch parameters (bucket_bits,
 * register_bits, seed) and the termination rule, exactly as in the
 * reference (README.md:117-120). */
typedef struct {
  uint32_t bucket_bits;       /* b, m = 2^b registers (default 7) */
  uint32_t register_bits;     /* r; 0 = 5 below 2^32 nodes, else 6 (engine.hpp:79-80) */
  uint64_t seed;              /* hash seed */
  uint32_t threads;           /* CPU scheduling knob; accepted and ignored */
  uint64_t task_size;         /* CPU scheduling knob; accepted and ignored */
  double systolic_threshold;  /* (0, 1], default 0.25 */
  int32_t termination;        /* 0 stabilisation, 1 threshold */
  double eps_inc;             /* threshold mode: relative increment floor */
  uint64_t max_iterations;    /* 0 = n + 1 */
  int32_t spill_to_disk;      /* accepted and ignored: HBM holds both generations */
  int32_t track_modified;     /* skip unmodified successors (time only) */
  int32_t use_systolic;       /* worklist bookkeeping (time only) */
  /* --- B200 options ---------------------------------------------------- */
  int32_t device;             /* CUDA device ordinal (default 0) */
  int32_t exact_sum;          /* 1 (default): N(t) total summed on the host in the
                                 reference's order -> bit-identical to
                                 engine.hpp:115-117; 0: deterministic device tree */
  uint64_t shard_begin;       /* node range [shard_begin, shard_end) this engine */
  uint64_t shard_end;         /* updates; (0, 0) = all nodes (single GPU) */
  uint32_t shard_count;       /* shards of the run (0: unknown).  With the peer-push
                                 exchange, equal shards of a graph whose counters
                                 exceed L2 and whose ids lack locality are
                                 relabelled by degree, interleaved across the
                                 shards (balanced arcs, hot rows first in each) */
  uint32_t expected_runs;     /* (new) runs the caller plans on this engine (multirun,
                                 main.cpp:263-283: hanf_reseed between them); 0 =
                                 unknown.  Only schedules depend on it: from 20 runs
                                 a large relabelled engine builds its source-blocked
                                 dense sweeps at create (see hanf_block_stats);
                                 otherwise they are built once the engine has run
                                 enough dense steps to repay the build */
} hanf_config;

/* IterationReport (engine.hpp:48-51) */
typedef struct {
  double sum;
  uint64_t modified;
} hanf_iteration_report;

/* SketchParams (hll.hpp:36-70) */
typedef struct {
  uint32_t bucket_bits;
  uint32_t registers;
  uint32_t register_bits;
  uint32_t words_per_counter; /* W = ceil(m*r/64), hll.hpp:58-60 */
  double alpha;               /* hll.hpp:27-34 */
  uint64_t seed;
} hanf_sketch_params;

/* ---- configuration ------------------------------------------------------ */
/* EngineConfig{} defaults (engine.hpp:32-46) + B200 defaults. */
hanf_status hanf_config_init(hanf_config* cfg);
/* SketchParams::make (hll.hpp:43-56): validates b in [4,20], r in [5,8]. */
hanf_status hanf_sketch_params_make(uint32_t bucket_bits, uint64_t seed,
                                    uint32_t register_bits,
                                    hanf_sketch_params* out);

/* ---- engine lifecycle ------------------------------------------------- */
/* NfEngine::NfEngine(const Graph&, EngineConfig) (engine.hpp:70-90):
 * validates the config, uploads the CSR to HBM, seeds counter v with item
 * v under `seed` (engine.hpp:84-85) on the device. */
hanf_status hanf_create(const hanf_graph_view* graph, const hanf_config* cfg,
                        hanf_engine** out);
void hanf_destroy(hanf_engine* engine);
/* (new) One engine over several GPUs of this process,
 * driven by one host thread - the reference keeps its parallelism inside
 * NfEngine::step (engine.hpp:157, parallel.hpp:16-48) and so does this
 * handle.  Nodes are split into `count` contiguous ranges (multiples of 64),
 * one shard engine per devices[k] (repeats allowed), attached to each other
 * for the peer-push exchange (peer access enabled between distinct
 * devices): each step, every shard's union kernels store the rows they
 * write into all peers' next generation over NVLink, the shards' streams
 * wait on each other's compute events (a device-side barrier, no host
 * round trip), and each shard commits the full arrays.  The handle accepts
 * hanf_step, hanf_step_launch / _complete, hanf_run_to_stabilisation,
 * hanf_sum_estimates, hanf_read_counters, hanf_save_counters, hanf_reset,
 * hanf_reseed, the accessors and hanf_destroy; results are bit-identical
 * to hanf_create's.  count in [1, HANF_MAX_PEERS + 1]; graphs with fewer
 * than 64 * count nodes get one shard. */
hanf_status hanf_create_multi(const hanf_graph_view* graph, const hanf_config* cfg,
                              const int32_t* devices, uint32_t count, hanf_engine** out);
/* (new) `runs` independent runs in one engine, run k under
 * seeds[k] (main.cpp:263-283 multirun): the graph is lifted to `runs`
 * copies (row v*runs + k) so one gather serves a node's runs together.
 * runs in {2, 4, 8} (1: hanf_create with seeds[0]); n * runs < 2^32; not
 * sharded.  Drive it with hanf_run_batch (hanf_step and the single-run
 * calls return HANF_INVALID_ARGUMENT). */
hanf_status hanf_create_batch(const hanf_graph_view* graph, const hanf_config* cfg,
                              const uint64_t* seeds, uint32_t runs, hanf_engine** out);
/* run_to_stabilisation (engine.hpp:233-275) of every run: run k's N(t)
 * and modified counts at values/modified[k*cap + t], t < lengths[k];
 * HANF_CAPACITY (lengths set) when a run needs more than cap. */
hanf_status hanf_run_batch(hanf_engine* engine, double* values, uint64_t* modified,
                           uint64_t cap, uint64_t* lengths);
/* Re-seeds the counters and rewinds to iteration 0 (a fresh NfEngine on
 * the same graph, without re-uploading it). */
hanf_status hanf_reset(hanf_engine* engine);
/* (new) hanf_reset under another HLL seed: the next run of a multi-seed
 * experiment (main.cpp:263-283 runs estimate_nf for seeds base + i) reuses
 * the uploaded graph, its task layout and its step graphs. */
hanf_status hanf_reseed(hanf_engine* engine, uint64_t seed);

/* Exact neighbourhood function (oracle.hpp:38-104): values[t] = ordered
 * pairs at distance <= t, t = 0..diameter, computed on GPU `device` as
 * bitset balls over batches of 2048 targets (hanf_exact.cu).  The same
 * guard as the reference's OracleGuard (max_nodes, max_work = n * arcs)
 * raises HANF_GUARD; HANF_CAPACITY when cap < the length (*len set). */
hanf_status hanf_exact_nf(const hanf_graph_view* graph, int32_t device, uint64_t max_nodes,
                          uint64_t max_work, uint64_t* values, uint64_t cap, uint64_t* len);

/* HCA1 counter snapshots (hll.hpp:241-305): the current counters written
 * byte for byte as the reference's save_counters writes them.  restore
 * loads a snapshot with the engine's (b, r, n, seed) into both generations
 * and resumes at `iteration` with every counter marked modified (the next
 * step recomputes every node: exact, whatever the snapshot's history);
 * HANF_PARSE_ERROR / HANF_IO_ERROR / HANF_INVALID_ARGUMENT on a bad or
 * mismatched file. */
hanf_status hanf_save_counters(hanf_engine* engine, const char* path);
hanf_status hanf_restore_counters(hanf_engine* engine, const char* path, uint64_t iteration);

/* ---- the hot path -------------------------------------------------------- */
/* (new) hanf_step split at the device boundary: launch enqueues the whole
 * step on the engine stream (hanf_stream) and returns at once; complete
 * waits for it and fills the report.  Lets a caller bracket exactly the
 * step's device work with its own stream events. */
hanf_status hanf_step_launch(hanf_engine* engine);
hanf_status hanf_step_complete(hanf_engine* engine, hanf_iteration_report* report);
/* NfEngine::sum_estimates() (engine.hpp:100-118). */
hanf_status hanf_sum_estimates(hanf_engine* engine, double* sum);
/* NfEngine::step() (engine.hpp:122-228): one iteration; counters become
 * the register-wise max over each node and its successors. */
hanf_status hanf_step(hanf_engine* engine, hanf_iteration_report* report);
/* NfEngine::run_to_stabilisation() (engine.hpp:233-275).  values/modified
 * receive N(0..T) and modified(0..T) (T+1 entries, clamped non-decreasing);
 * HANF_CAPACITY if capacity < T+1 (length still reports T+1);
 * HANF_GUARD when the iteration cap is exceeded. */
hanf_status hanf_run_to_stabilisation(hanf_engine* engine, double* values,
                                      uint64_t* modified, uint64_t capacity,
                                      uint64_t* length, double* wall_seconds);
/* Copies the N(t)/modified vectors of the last run_to_stabilisation (the
 * engine keeps them, so a HANF_CAPACITY result can be fetched in full). */
hanf_status hanf_last_result(const hanf_engine* engine, double* values,
                             uint64_t* modified, uint64_t capacity,
                             uint64_t* length);
/* estimate_nf(const Graph&, const EngineConfig&) (engine.hpp:295-298). */
hanf_status hanf_estimate_nf(const hanf_graph_view* graph, const hanf_config* cfg,
                             double* values, uint64_t* modified,
                             uint64_t capacity, uint64_t* length,
                             double* wall_seconds);

/* ---- accessors ----------------------------------------------------------- */
/* NfEngine::counters() (engine.hpp:94) -> CounterArray::data() (hll.hpp:224):
 * copies counters [first, first+count) in the reference packing (W u64
 * words each) to dst.  HANF_OUT_OF_RANGE past n. */
hanf_status hanf_read_counters(hanf_engine* engine, uint64_t first,
                               uint64_t count, uint64_t* dst);
hanf_status hanf_params(const hanf_engine* engine, hanf_sketch_params* out); /* :92 */
hanf_status hanf_iteration(const hanf_engine* engine, uint64_t* t);          /* :95 */
hanf_status hanf_systolic_active(const hanf_engine* engine, int32_t* active); /* :96 */
hanf_status hanf_num_nodes(const hanf_engine* engine, uint64_t* n);
/* Thread-local message of the last failing call on this thread. */
const char* hanf_last_error(void);

/* ---- device plumbing (bench, multi-GPU orchestration) -------------------- */
/* cudaStream_t the engine launches on (as void*). */
hanf_status hanf_stream(const hanf_engine* engine, void** stream);
/* Kernels launched by this engine since creation. */
hanf_status hanf_launch_count(const hanf_engine* engine, uint64_t* launches);
/* Source-blocked dense sweeps (an engine-internal schedule of
 * NfEngine::step's union loop, engine.hpp:157-185; results are unchanged):
 * the number of (successor segment, source) items and the arcs they cover,
 * 0 / 0 while the engine sweeps every arc from its own node's list.  Built
 * for large relabelled engines: at create when hanf_config.expected_runs >= 20,
 * else at the hanf_reset / hanf_reseed that follows the engine's 96th dense
 * step, when the steps saved so far would have repaid the build
 * (HANF_BLOCK=1: at create, 2: at the first reset whatever the size, 0: never). */
hanf_status hanf_block_stats(const hanf_engine* engine, uint64_t* items, uint64_t* arcs);
/* Phase timing with CUDA events on the engine stream (off by default):
 * union sweep (union + hub kernels), estimates + block sums, totals.
 * Accumulated over the steps since the last hanf_set_timing(e, 1). */
hanf_status hanf_set_timing(hanf_engine* engine, int32_t enable);
hanf_status hanf_timing(const hanf_engine* engine, double* union_ms,
                        double* estimate_ms, double* reduce_ms, uint64_t* steps);
/* Device buffers of the engine, for collectives over the node shards. */
typedef struct {
  void* next_counters;     /* u64[n*row_pitch]: the generation being written by step */
  void* next_modified;     /* u64[ceil(n/64)] bitmap of counters changed by step */
  void* block_sums;        /* f64[ceil(n/64)] per-64-counter estimate sums */
  uint64_t words_per_counter;
  uint64_t blocks;         /* ceil(n/64) */
  uint64_t shard_begin, shard_end; /* node range updated by this engine */
  uint64_t row_pitch;      /* u64 words between consecutive counters (>= W) */
  uint32_t relabelled;     /* rows are renumbered by degree (counters of row r are
                              node order[r]'s; hanf_read_counters undoes it) */
  uint32_t reserved;
} hanf_buffers;
hanf_status hanf_device_buffers(hanf_engine* engine, hanf_buffers* out);
/* Sharded step, phase 1: compute this engine's node range into the next
 * generation (device-side; returns immediately, stream-ordered). */
hanf_status hanf_shard_compute(hanf_engine* engine);
/* (new) Changed-rows exchange for sharded steps: after hanf_shard_compute,
 * pack writes to the device buffers ids[cap] / rows[cap * row_pitch] the
 * rows of this engine's range that the step wrote (changed, or stale:
 * changed by the previous step).  Those are exactly the rows in which the
 * peers' copies of the next generation differ, so peers that unpack every
 * other shard's packet (instead of receiving whole shards) hold the same
 * next generation.  HANF_CAPACITY (count set) when more than cap rows.
 * ids >= n in a packet are padding. */
hanf_status hanf_shard_pack(hanf_engine* engine, uint32_t* ids, uint64_t* rows, uint64_t cap,
                            uint64_t* count);
hanf_status hanf_shard_unpack(hanf_engine* engine, const uint32_t* ids, const uint64_t* rows,
                              uint64_t count);
/* Sharded step, phase 2 (after the next-generation shards, modified bitmap
 * and block sums of every rank have been exchanged into this engine's
 * buffers): swap generations and produce the IterationReport. */
hanf_status hanf_shard_commit(hanf_engine* engine, hanf_iteration_report* report);
/* (new) Peer-push exchange: the fused alternative to the collectives above
 * (replaces the per-iteration all-gather of SURVEY 8(e); the reference has
 * no distributed path).  Every shard engine keeps its two counter
 * generations, both modified bitmaps and two block-sum inboxes in one
 * IPC-exportable device arena of identical layout on every rank.  Once the
 * engines are attached to each other, hanf_shard_compute's union and
 * worklist kernels store every row they write (changed, or stale) into the
 * peers' next generation as well - over NVLink peer memory, tile by tile
 * as the rows are produced - and a last kernel publishes the shard's
 * modified-bitmap words and block sums into the peers' arenas.  One step is
 * then: hanf_shard_compute; wait for the engine stream; a barrier across
 * the ranks; hanf_shard_commit.  No counter bytes pass through a
 * collective; rows that did not change are never sent (the tail iterations
 * move kilobytes).  Block sums are double-buffered by generation, so a
 * rank may start step t+1 while a slower peer is still committing step t.
 * Needed-rows filter: each engine derives from its task-ordered successor
 * array the rows its nodes can ever gather (n bits, in the arena); attach
 * copies every peer's bits over this shard's range, and a written row is
 * pushed only to the peers that gather it (about 44% of the pushes of a
 * relabelled R-MAT at 8 shards).  A peer's copies of rows it never
 * gathers go stale; hanf_read_counters / hanf_save_counters first copy
 * every peer's own range of the current generation back (peer memory).
 * HANF_PEER_NEED=0 (environment, read at create) pushes every row. */
typedef struct {
  uint8_t ipc_handle[64];  /* cudaIpcMemHandle_t of the exchange arena */
  uint64_t arena_bytes;
  uint64_t n, row_pitch;
  uint64_t shard_begin, shard_end;
  int32_t device;
  int32_t relabelled;      /* bit 0: relabelled shards (hanf_config.shard_count), all or
                              none; bit 1: byte-layout counter rows (all or none) */
} hanf_shard_peer;
#define HANF_MAX_PEERS 7
/* Describes this shard engine's arena for the other ranks. */
hanf_status hanf_shard_export(hanf_engine* engine, hanf_shard_peer* out);
/* Opens the other ranks' arenas (cudaIpcOpenMemHandle; peers[self] is this
 * engine's own export and is not opened).  The ranges must tile [0, n) and
 * the layouts must agree; at most HANF_MAX_PEERS peers. */
hanf_status hanf_shard_attach(hanf_engine* engine, const hanf_shard_peer* peers, uint32_t count,
                              uint32_t self);
/* Same, for shard engines of one process (device pointers used directly:
 * same device, or peer access enabled by the caller). */
hanf_status hanf_shard_attach_local(hanf_engine* engine, hanf_engine* const* peers, uint32_t count,
                                    uint32_t self);
/* Relabelled shards (hanf_config.shard_count) under the peer-push
 * exchange, optional: after the compute barrier, re-sums this rank's
 * 1/shard_count slice of the original-id blocks from the pushed estimates
 * and publishes it to every rank; after a second barrier hanf_shard_commit
 * only totals them.  Without it every rank re-sums every block in its
 * commit (n estimate gathers per rank per dense step).  A no-op for other
 * engines. */
hanf_status hanf_shard_reduce(hanf_engine* engine);
/* Waits for this engine's enqueued device work (hanf_shard_compute's
 * pushes included): the step's barrier across the ranks comes after it. */
hanf_status hanf_shard_wait(hanf_engine* engine);
/* (new) Peer-push traffic of the last committed step, for reporting:
 * *changed = rows of this shard's range the step changed, *pushed = the
 * row stores those changes sent to peers (sum over peers of the changed
 * rows each peer gathers; changed * peers without the needed-rows filter).
 * Stale rows rewritten with them are pushed under the same filter. */
hanf_status hanf_shard_push_stats(hanf_engine* engine, uint64_t* changed, uint64_t* pushed);
/* Back to the collective exchange (closes opened IPC mappings). */
hanf_status hanf_shard_detach(hanf_engine* engine);

/* ---- stats.hpp (host arithmetic on N(t)) ---------------------------------- */
/* cdf_from_nf + distribution_from_cdf (stats.hpp:33-60). */
hanf_status hanf_distance_distribution(const double* nf, uint64_t length,
                                       double* mean, double* variance,
                                       double* spid);
/* effective_diameter (stats.hpp:65-77). */
hanf_status hanf_effective_diameter(const double* nf, uint64_t length,
                                    double alpha, int32_t interpolated,
                                    double* out);

/* ---- graphs: CSR construction, generators, HBG1 ----------------------------- */
/* Graph::from_edges (graph.hpp:29-44): sort + dedupe; ids must be < n. */
hanf_status hanf_graph_from_edges(uint64_t n, const uint32_t* src,
                                  const uint32_t* dst, uint64_t count,
                                  hanf_graph** out);
/* Reference fixtures: gen_uniform_random (graph.hpp:262-285) and
 * gen_clique_path (graph.hpp:238-258), same bits. */
hanf_status hanf_gen_uniform_random(uint64_t n, double d, uint64_t seed,
                                    hanf_graph** out);
hanf_status hanf_gen_clique_path(uint64_t k, uint64_t l, hanf_graph** out);
/* BASELINE.json synthetic configs. */
hanf_status hanf_gen_erdos_renyi(uint64_t n, double mean_degree, uint64_t seed,
                                 hanf_graph** out);
hanf_status hanf_gen_rmat(uint32_t scale, uint32_t edge_factor, double a,
                          double b, double c, uint64_t seed,
                          uint64_t permute_seed, hanf_graph** out);
hanf_status hanf_gen_copying(uint64_t n, double exponent, double mean_degree,
                             uint64_t max_degree, double copy_prob,
                             uint64_t window, uint64_t seed, hanf_graph** out);
hanf_status hanf_gen_barabasi_albert(uint64_t n, uint32_t m, uint64_t seed,
                                     uint64_t permute_seed, hanf_graph** out);
/* (new) The same graphs built on GPU `device` with device
 * radix sorts: Graph::from_edges (graph.hpp:29-44) and the R-MAT generator,
 * bit-identical CSR to hanf_graph_from_edges / hanf_gen_rmat, returned in
 * host memory.  HANF_CUDA_ERROR without a device. */
hanf_status hanf_graph_from_edges_gpu(int32_t device, uint64_t n, const uint32_t* src,
                                      const uint32_t* dst, uint64_t count, hanf_graph** out);
hanf_status hanf_gen_rmat_gpu(int32_t device, uint32_t scale, uint32_t edge_factor, double a,
                              double b, double c, uint64_t seed, uint64_t permute_seed,
                              hanf_graph** out);
/* transpose (graph.hpp:72-84). */
hanf_status hanf_graph_transpose(const hanf_graph* g, hanf_graph** out);
/* HBG1 CSR cache (graph.hpp:178-218, FORMATS.md:13-23). */
hanf_status hanf_graph_save_csr(const hanf_graph* g, const char* path);
hanf_status hanf_graph_load_csr(const char* path, hanf_graph** out);
hanf_status hanf_graph_view_of(const hanf_graph* g, hanf_graph_view* view);
void hanf_graph_free(hanf_graph* g);

/* (new: the reference keeps graphs in pageable vectors) Page-locks the host
 * range [p, p + bytes) in place (cudaHostRegister) so hanf_create uploads
 * it by DMA at full link rate instead of through a bounce buffer; pair
 * with hanf_unpin_host before the memory is freed.  Large allocations made
 * with transparent huge pages (numpy, or madvise(MADV_HUGEPAGE)) register
 * as few IOMMU mappings and reach ~55 GB/s H2D on B200 hosts
 * (profiles/r01_h2d.md). */
hanf_status hanf_pin_host(const void* p, uint64_t bytes);
hanf_status hanf_unpin_host(const void* p);

#ifdef __cplusplus
}
#endif
#endif /* HANF_H */
