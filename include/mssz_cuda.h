/* mssz_cuda.h — C-ABI of the B200-native MSz segmentation-correction loop.
 *
 * Drop-in boundary for the reference's hot path.  The reference exposes C++
 * templates with no FFI layer; every entry point below replaces
 * one of them with plain pointers and sizes:
 *
 *   mssz_cu_derive_edits_{f32,f64}
 *       replaces  template<class T> EditSet<T> derive_edits(const GridTopology&,
 *                   const T* original, const T* decompressed, double xi,
 *                   const DeriveOptions<T>& = {}, EditStats* = nullptr)
 *                 /root/reference/proj/core/include/mssz/edit_engine.hpp:183-186
 *                 (implementation edit_engine.cpp:386-435).  Host buffers in,
 *                 callee-allocated EditSet out (release with mssz_cu_free).
 *   mssz_cu_derive_edits_into_{f32,f64}
 *       same, caller-provided host output buffers (no allocation per call).
 *   mssz_cu_derive_edits_device_{f32,f64}
 *       same, device-resident inputs/outputs on a caller stream.
 *   mssz_cu_compute_directions_{f32,f64}
 *       replaces  compute_directions<T> (mss.hpp:44-50, mss.cpp:11-30); returns
 *                 the reference's u64 asc/desc vertex ids.
 *   mssz_cu_compute_labels
 *       replaces  compute_labels (mss.hpp:58-60, mss.cpp:84-97).
 *   mssz_cu_classify_critical
 *       replaces  classify_critical (mss.hpp:52, mss.cpp:40-47).
 *   mssz_cu_detect_false_critical_{f32,f64}
 *       replaces  EditState<T>::detect_false_critical (edit_engine.hpp:100,
 *                 edit_engine.cpp:134-158) for an (original, edited) pair.
 *   mssz_cu_lower_step_{f32,f64}, mssz_cu_representable_floor_{f32,f64}
 *       element-wise EditState<T>::lower_step (edit_engine.cpp:75-86) and
 *       representable_floor (edit_engine.cpp:22-29).
 *   mssz_cu_apply_edits_{f32,f64}
 *       replaces  apply_edits<T> (edit_engine.hpp:188-190, edit_engine.cpp:437-450);
 *                 indices are applied in order (a repeated index: the last value
 *                 wins); an out-of-range index fails with corrupt_archive and
 *                 writes no output.
 *   mssz_cu_r_targets_{f32,f64}
 *       one R-loop batch's target set behind the R gate (a pair with false
 *                 critical points returns 0 targets, as run_r_loop returns at
 *                 edit_engine.cpp:338) (run_r_loop, edit_engine.cpp:336-352:
 *                 collect_mismatched + find_troublemaker :293-315 + claim) for an
 *                 (original, edited) pair, computed by the engine's tiled pass
 *                 (mode 0) or its sparse Up(X) pass (mode 1).  targets: caller
 *                 buffer of n entries, sorted, distinct.  info = {false critical
 *                 points of the pair (the R gate, :338), divergent mismatched
 *                 (vertex, family) pairs = distinct troublemaker sources v_i,
 *                 path used (0 tiled, 1 sparse; mode 1 falls back to 0 when
 *                 Up(X) is too large)}.  Parity harness entry point.
 *
 * Conventions (mirroring errors.hpp:9-16): every function returns 0 or the
 * reference ErrKind value (2 usage, 3 io, 4 bound_violation, 5 non_convergence,
 * 6 corrupt_archive, 7 internal) and sets a thread-local message readable with
 * mssz_cu_last_error().  99 = CUDA runtime failure (no device, launch error).
 * Grids are row-major with axis 0 fastest (grid.hpp:32-43); dims[2] is
 * ignored when ndims == 2.  Vertex counts must be < 2^32 - 1 (device ids are
 * u32; the reference caps at 2^40, grid.cpp:19 — larger grids are sharded).
 * Calls are synchronous and blocking, like the reference.  There is NO CPU
 * fallback: without a usable CUDA device every compute entry point fails with 99.
 */
#ifndef MSSZ_CUDA_H
#define MSSZ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSSZ_CU_OK 0
#define MSSZ_CU_ERR_USAGE 2
#define MSSZ_CU_ERR_IO 3
#define MSSZ_CU_ERR_BOUND_VIOLATION 4
#define MSSZ_CU_ERR_NON_CONVERGENCE 5
#define MSSZ_CU_ERR_CORRUPT_ARCHIVE 6
#define MSSZ_CU_ERR_INTERNAL 7
#define MSSZ_CU_ERR_CALLBACK 98 /* on_batch returned nonzero: the correction was abandoned */
#define MSSZ_CU_ERR_CUDA 99

/* Mirrors DeriveOptions<T> (edit_engine.hpp:70-82).  ExecPolicy becomes a
 * device choice; on_batch becomes an optional host callback (debug/parity
 * mode: the device loop then stops after every batch so the host can read g).
 * In the reference an exception thrown by on_batch aborts derive_edits; here the
 * callback returns nonzero to abort, and the call returns MSSZ_CU_ERR_CALLBACK
 * (the language bindings re-raise the callback's own exception).
 * on_batch_mode: MSSZ_CU_ON_BATCH_EVERY (0) = after every fix batch, exactly the
 * reference's call sites (edit_engine.cpp:275, :364); MSSZ_CU_ON_BATCH_PHASES (1)
 * = only after each complete C pass (all four subloops, :280-291) and after
 * each R iteration, with the device loop running at full speed in between
 * (snapshots of large fields for parity checks). */
typedef struct mssz_cu_options {
  uint64_t outer_cap;   /* default 1000 */
  uint64_t subloop_cap; /* default 640, per run_subloop invocation */
  uint64_t r_cap;       /* default 100000, per run_r_loop invocation */
  int32_t force;        /* accept |f - fhat| > xi inputs */
  int32_t device;       /* CUDA ordinal; -1 = current device */
  int (*on_batch)(const void* g_host, uint64_t n, void* user); /* NULL = off; nonzero = abort */
  void* on_batch_user;
  int32_t profile; /* CUDA-event kernel timing into stats.kernel_ms: bit 0 = every class,
                      bit (c + 1) = class c only (MSSZ_CU_PROF_*) */
  int32_t on_batch_mode; /* MSSZ_CU_ON_BATCH_EVERY / MSSZ_CU_ON_BATCH_PHASES */
} mssz_cu_options;

#define MSSZ_CU_ON_BATCH_EVERY 0
#define MSSZ_CU_ON_BATCH_PHASES 1

/* Inside an on_batch callback: what the snapshot is.  out = {kind, outer
 * iteration (1-based), index (1-based C pass, or R iteration, within that outer
 * iteration; for kind BATCH the C pass in progress)}. */
#define MSSZ_CU_PHASE_BATCH 0       /* a C fix batch (mode EVERY) */
#define MSSZ_CU_PHASE_C_PASS 1      /* a complete C pass (mode PHASES) */
#define MSSZ_CU_PHASE_R_ITERATION 2 /* an R iteration (both modes) */
int mssz_cu_batch_phase(uint64_t out[3]);

/* kernel classes of mssz_cu_stats.kernel_ms / kernel_count */
#define MSSZ_CU_PROF_VALIDATE 0
#define MSSZ_CU_PROF_DIRECTIONS 1
#define MSSZ_CU_PROF_DETECT_KIND 2
#define MSSZ_CU_PROF_DETECT_ALL 3
#define MSSZ_CU_PROF_SUBLOOP 4
#define MSSZ_CU_PROF_LABEL_INIT 5 /* tiled label pass (k_label_tile) */
#define MSSZ_CU_PROF_LABEL_JUMP 6 /* pointer jumping (exits / generic API) */
#define MSSZ_CU_PROF_RFIX 7
#define MSSZ_CU_PROF_FRONTIER 8
#define MSSZ_CU_PROF_COMPACT 9
#define MSSZ_CU_PROF_LABEL_FINISH 10
#define MSSZ_CU_PROF_FIX 11 /* host-driven huge batch: fix_list */
#define MSSZ_CU_PROF_SPARSE 12 /* sparse R iteration kernels */
#define MSSZ_CU_PROF_DETECT_DIRTY 13 /* subloop detection over changed chunks (k_detect_dirty) */
#define MSSZ_CU_PROF_CLASSES 16

/* Mirrors EditStats (edit_engine.hpp:54-68) field for field, then adds the
 * device-side timings/counters of the B200 engine. */
typedef struct mssz_cu_stats {
  uint64_t outer_iterations;
  uint64_t c_passes;
  uint64_t sub_iterations[4]; /* FPmax, FPmin, FNmax, FNmin */
  uint64_t r_iterations;
  uint64_t effective_edits;
  uint64_t touched;
  uint64_t input_bound_violations;
  double direction_seconds; /* device time of full direction sweeps (CUDA events) */
  double label_seconds;     /* device time of label passes (CUDA events) */
  /* B200 extras */
  double h2d_seconds;
  double d2h_seconds;
  double device_seconds; /* whole device-side correction, validation to compaction */
  uint64_t label_passes;
  uint64_t label_rounds;
  uint64_t detect_sweeps;
  uint64_t frontier_vertices; /* sum over batches of |S ∪ N(S)| re-evaluated */
  uint64_t kernel_launches;   /* kernels launched by this call */
  uint64_t big_batches;       /* C batches run grid-wide inside the persistent kernel */
  uint64_t huge_batches;      /* C batches run by host-launched streaming kernels */
  uint64_t label_tiles;       /* label tiles re-resolved (phase 1) over all label passes */
  uint64_t rfix_tiles;        /* label tiles whose mismatch bits were recomputed */
  uint64_t sparse_iterations; /* R iterations resolved by the sparse Up(X) pass */
  uint64_t sparse_up;         /* sum of |Up(X)| over sparse passes */
  uint64_t rfix_divergent;    /* (vertex, family) pairs k_rfix_tiles resolved a label for */
  uint64_t subloop_items;     /* worklist items fixed by the persistent C-loop kernel */
  uint64_t subloop_edits;     /* edits applied by the persistent C-loop kernel (its batches) */
  uint64_t skipped_subloops;  /* subloops skipped without a launch (list provably empty) */
  uint64_t kernel_count[MSSZ_CU_PROF_CLASSES]; /* launches per kernel class */
  double kernel_ms[MSSZ_CU_PROF_CLASSES];      /* device ms per profiled class */
} mssz_cu_stats;

void mssz_cu_default_options(mssz_cu_options* opt);
const char* mssz_cu_last_error(void);
void mssz_cu_free(void* p);
int mssz_cu_device_count(void);
const char* mssz_cu_version(void);
/* Frees the cached per-device workspace (device buffers, pinned staging). */
int mssz_cu_release_workspace(int device);

#define MSSZ_CU_DECLARE_TYPED(SUF, T)                                                         \
  int mssz_cu_derive_edits_##SUF(int ndims, const uint64_t* dims, const T* original,          \
                                 const T* decompressed, double xi, const mssz_cu_options* opt, \
                                 uint64_t** indices_out, T** values_out, uint64_t* count_out,  \
                                 mssz_cu_stats* stats_out);                                    \
  int mssz_cu_derive_edits_into_##SUF(int ndims, const uint64_t* dims, const T* original,     \
                                      const T* decompressed, double xi,                        \
                                      const mssz_cu_options* opt, uint64_t* indices,           \
                                      T* values, uint64_t capacity, uint64_t* count_out,       \
                                      mssz_cu_stats* stats_out);                               \
  int mssz_cu_derive_edits_device_##SUF(int ndims, const uint64_t* dims,                      \
                                        const T* d_original, const T* d_decompressed,          \
                                        double xi, const mssz_cu_options* opt,                 \
                                        uint64_t* d_indices, T* d_values, uint64_t capacity,   \
                                        uint64_t* count_out, mssz_cu_stats* stats_out,         \
                                        void* cuda_stream);                                    \
  int mssz_cu_compute_directions_##SUF(int ndims, const uint64_t* dims, const T* values,      \
                                       uint64_t* asc, uint64_t* desc);                         \
  int mssz_cu_compute_direction_codes_##SUF(int ndims, const uint64_t* dims, const T* values, \
                                            uint8_t* codes);                                   \
  int mssz_cu_detect_false_critical_##SUF(int ndims, const uint64_t* dims, const T* original, \
                                          const T* edited, uint64_t counts[4],                 \
                                          uint64_t* lists);                                    \
  int mssz_cu_detect_kind_##SUF(int ndims, const uint64_t* dims, const T* original,           \
                                const T* edited, int kind, uint64_t* list,                     \
                                uint64_t* count_out);                                          \
  int mssz_cu_lower_step_##SUF(uint64_t n, const T* g, const T* f, double xi, T* g_out,       \
                               uint8_t* moved);                                                \
  int mssz_cu_representable_floor_##SUF(uint64_t n, const T* f, double xi, T* out);           \
  int mssz_cu_apply_edits_##SUF(uint64_t n, const T* decompressed, const uint64_t* indices,   \
                                const T* values, uint64_t count, T* out);                     \
  int mssz_cu_r_targets_##SUF(int ndims, const uint64_t* dims, const T* original,              \
                              const T* edited, int mode, uint64_t* targets, uint64_t* count,   \
                              uint64_t info[3]);

MSSZ_CU_DECLARE_TYPED(f32, float)
MSSZ_CU_DECLARE_TYPED(f64, double)

/* asc/desc/labels are the reference's u64 vertex ids (mss.hpp:24-42). */
int mssz_cu_compute_labels(int ndims, const uint64_t* dims, const uint64_t* asc,
                           const uint64_t* desc, uint64_t* max_label, uint64_t* min_label);
/* maxima/minima: caller buffers of n entries; counts out; sorted ascending. */
int mssz_cu_classify_critical(uint64_t n, const uint64_t* asc, const uint64_t* desc,
                              uint64_t* maxima, uint64_t* n_max, uint64_t* minima,
                              uint64_t* n_min);

/* ---- z-slab sharding ----------------------------------------
 * A 3D field is split along axis 2 into P contiguous slabs of >= 2 planes
 * (slab r owns planes [floor(Z r/P), floor(Z (r+1)/P))).  Each rank passes its
 * WINDOW: the owned planes plus up to two halo planes per side, i.e. planes
 * [wz0, wz1) of mssz_cu_slab_range().  The edits a rank returns are the ones in
 * its owned planes, as GLOBAL ids, sorted; concatenated in rank order they are
 * the EditSet of derive_edits (edit_engine.cpp:368-378) on the whole field, and
 * the result -- edits, values and EditStats -- is identical to the
 * single-device engine's.  Global ids are u64: the whole field may hold up to
 * the reference's 2^40 vertices (grid.cpp:19); a z plane and each rank's
 * window must stay below 2^32 - 1 vertices (device-local ids are u32).
 *
 * One process per GPU: rank 0 calls mssz_cu_comm_unique_id and broadcasts the
 * id (e.g. torch.distributed), then every rank calls mssz_cu_comm_init
 * (NCCL: all-gathers of per-batch status records and boundary label tables,
 * send/recv of boundary edits with the z neighbours). */
#define MSSZ_CU_UNIQUE_ID_BYTES 128
typedef struct mssz_cu_comm mssz_cu_comm;

/* out = {z0, z1, wz0, wz1}: owned planes [z0, z1), window planes [wz0, wz1). */
int mssz_cu_slab_range(uint64_t Z, int nranks, int rank, uint64_t out[4]);
int mssz_cu_comm_unique_id(uint8_t* id /* MSSZ_CU_UNIQUE_ID_BYTES */);
int mssz_cu_comm_init(const uint8_t* id, int nranks, int rank, int device, mssz_cu_comm** out);
int mssz_cu_comm_destroy(mssz_cu_comm* comm);

/* _slab: host window in, this slab's part of the EditSet out (offset_out = its
 *   position in the global EditSet); stats are global (identical on every rank).
 * _slab_device: same, device-resident window and outputs, ordered after cuda_stream.
 * _slabs_local: nslabs virtual ranks in this process (host threads on
 *   devices[r % ndevices], or the current device); whole-field host buffers in,
 *   whole EditSet out (single-GPU testing of the sharded schedule). */
#define MSSZ_CU_DECLARE_SLAB(SUF, T)                                                              \
  int mssz_cu_derive_edits_slab_##SUF(mssz_cu_comm* comm, int ndims, const uint64_t* dims,       \
                                      const T* original_window, const T* decompressed_window,   \
                                      double xi, const mssz_cu_options* opt, uint64_t* indices, \
                                      T* values, uint64_t capacity, uint64_t* count_out,        \
                                      uint64_t* offset_out, mssz_cu_stats* stats_out);          \
  int mssz_cu_derive_edits_slab_device_##SUF(                                                    \
      mssz_cu_comm* comm, int ndims, const uint64_t* dims, const T* d_original_window,           \
      const T* d_decompressed_window, double xi, const mssz_cu_options* opt, uint64_t* d_indices, \
      T* d_values, uint64_t capacity, uint64_t* count_out, uint64_t* offset_out,                 \
      mssz_cu_stats* stats_out, void* cuda_stream);                                              \
  int mssz_cu_derive_edits_slabs_local_##SUF(int nslabs, const int* devices, int ndevices,      \
                                             int ndims, const uint64_t* dims, const T* original, \
                                             const T* decompressed, double xi,                   \
                                             const mssz_cu_options* opt, uint64_t* indices,      \
                                             T* values, uint64_t capacity, uint64_t* count_out,  \
                                             mssz_cu_stats* stats_out);

MSSZ_CU_DECLARE_SLAB(f32, float)
MSSZ_CU_DECLARE_SLAB(f64, double)

/* ---- verification report: build_report, tools/mssz.cpp:84-104 ----
 * VerificationReport (metrics.hpp:14-23) field for field, then B200 extras.  The
 * reference CLI's `verify` exits 0 iff mss_distortion == 0 && bound_violations == 0
 * (tools/mssz.cpp:250).  psnr's sum of squares is a deterministic tree reduction
 * (reference: sequential), equal to 1e-12 relative; every count is exact. */
typedef struct mssz_cu_report {
  double mss_distortion;      /* label mismatches / N (metrics.cpp:12-15) */
  double right_labeled_ratio; /* 1 - mss_distortion */
  double psnr;                /* dB, +inf when rmse == 0 (metrics.cpp:18-32) */
  double edit_ratio;          /* edit_count / N */
  double ocr;                 /* original bytes / archive bytes (0 when archive_bytes == 0) */
  double obr;                 /* 8 * archive bytes / N */
  uint64_t bound_violations;  /* |f - g| > xi in double (metrics.cpp:46-56) */
  uint64_t fp_max, fp_min, fn_max, fn_min; /* first-match classes (tools/mssz.cpp:69-82) */
  /* B200 extras */
  uint64_t mismatches;
  double sum_sq, value_lo, value_hi;
  double device_seconds;
  uint64_t kernel_launches;
} mssz_cu_report;

#define MSSZ_CU_DECLARE_VERIFY(SUF, T)                                                              \
  int mssz_cu_verify_##SUF(int ndims, const uint64_t* dims, const T* original, const T* candidate,  \
                           double xi, uint64_t edit_count, uint64_t archive_bytes,                   \
                           const mssz_cu_options* opt, mssz_cu_report* out);                         \
  int mssz_cu_verify_device_##SUF(int ndims, const uint64_t* dims, const T* d_original,             \
                                  const T* d_candidate, double xi, uint64_t edit_count,              \
                                  uint64_t archive_bytes, const mssz_cu_options* opt,                \
                                  mssz_cu_report* out, void* cuda_stream);
MSSZ_CU_DECLARE_VERIFY(f32, float)
MSSZ_CU_DECLARE_VERIFY(f64, double)

/* The `mss` subcommand (tools/mssz.cpp:260-266): SegmentationLabels of a field,
 * compute_labels(compute_directions(values)) in one device pass; u64 max and min
 * labels (mss.hpp:37-42).  export_labels (mss.cpp:135-145) writes M then m as u64 LE. */
int mssz_cu_segmentation_f32(int ndims, const uint64_t* dims, const float* values, uint64_t* max_label,
                             uint64_t* min_label);
int mssz_cu_segmentation_f64(int ndims, const uint64_t* dims, const double* values, uint64_t* max_label,
                             uint64_t* min_label);

/* ---- base codec on the GPU: compress_base / decompress_base ----
 * compress: values -> reconstruction (the f-hat the correction loop takes) and the
 *   quantisation symbols (0 = escape, else 1 + zigzag(q)) that huffman::encode_stream
 *   codes (base_codec.cpp:76-120); literals are the values at symbol-0 positions in
 *   index order.  decompress: (symbols, literals) after huffman::decode_stream ->
 *   reconstruction (base_codec.cpp:122-152).  Bit-exact with the reference (Lorenzo
 *   order-1 prediction, double arithmetic, block wavefront).  device_ms (nullable):
 *   device time of the wavefront. */
int mssz_cu_compress_base_f32(int ndims, const uint64_t* dims, const float* values, double xi, float* recon,
                              uint32_t* symbols /* nullable */, uint64_t* escapes, double* device_ms);
int mssz_cu_compress_base_f64(int ndims, const uint64_t* dims, const double* values, double xi, double* recon,
                              uint32_t* symbols /* nullable */, uint64_t* escapes, double* device_ms);
int mssz_cu_decompress_base_f32(int ndims, const uint64_t* dims, const uint32_t* symbols, const float* literals,
                                uint64_t n_literals, double xi, float* recon, double* device_ms);
int mssz_cu_decompress_base_f64(int ndims, const uint64_t* dims, const uint32_t* symbols, const double* literals,
                                uint64_t n_literals, double xi, double* recon, double* device_ms);

/* ---- edit-set encoding: encode_edits<T>, edit_codec.cpp:188-222 ----
 * Byte-identical payload: u64 count, u64 index-stream length, index stream =
 * backend(huffman(rle(leb128(delta(indices))))), value stream = backend(raw LE
 * values); codec 0 = store, 1 = raw DEFLATE (zlib, as the reference).  Delta,
 * LEB128, RLE, the histogram and the bit packing run on the GPU; code lengths
 * and DEFLATE on the host.  Payload is callee-allocated (mssz_cu_free);
 * device_ms (nullable) = device time of the GPU stages. */
int mssz_cu_encode_edits_f32(const uint64_t* indices, const float* values, uint64_t count, int codec,
                             uint8_t** payload, uint64_t* payload_len, double* device_ms);
int mssz_cu_encode_edits_f64(const uint64_t* indices, const double* values, uint64_t count, int codec,
                             uint8_t** payload, uint64_t* payload_len, double* device_ms);

#ifdef __cplusplus
}
#endif
#endif /* MSSZ_CUDA_H */
