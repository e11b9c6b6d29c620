/* TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 correction loop.
 *
 * Plain-C restatement of the reference's hot path
 * (/root/reference/proj/core/src/{grid,mss,edit_engine}.cpp), used ONLY by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  The
 * product library (paper_2406_09423_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every entry point below against the
 * committed golden vectors in tests/golden/ (generated from the UNMODIFIED
 * reference via oracle/_ref/libmssz_ref.so by tests/golden/make_golden.py)
 * and, when oracle/_ref/libmssz_ref.so is present, against the reference
 * itself on seeded random inputs.
 *
 * Two fix schedules are provided for derive_edits:
 *   MSSZ_ORACLE_GAUSS_SEIDEL  the reference's serial schedule
 *                             (edit_engine.cpp:390-404: FPmin/FNmax targets are
 *                             g_argmax_neighbor on LIVE g, in list order)
 *   MSSZ_ORACLE_JACOBI        the B200 schedule: every batch's targets come
 *                             from the pre-batch snapshot (equal to
 *                             g_argmax_neighbor at batch start), so the result
 *                             is order-independent.  The GPU must match this
 *                             one bit-for-bit (edit set AND every EditStats
 *                             counter); the serial reference within the
 *                             tolerance stated in DESIGN.md.
 * Error codes are the reference ErrKind values (errors.hpp:9-16).
 */
#ifndef MSSZ_ORACLE_H
#define MSSZ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MSSZ_ORACLE_GAUSS_SEIDEL = 0, MSSZ_ORACLE_JACOBI = 1 };

typedef struct {
  uint64_t outer_cap;
  uint64_t subloop_cap;
  uint64_t r_cap;
  int force;
  int schedule; /* MSSZ_ORACLE_GAUSS_SEIDEL or MSSZ_ORACLE_JACOBI */
} mssz_oracle_options;

typedef struct {
  uint64_t outer_iterations;
  uint64_t c_passes;
  uint64_t sub_iterations[4]; /* FPmax, FPmin, FNmax, FNmin */
  uint64_t r_iterations;
  uint64_t effective_edits;
  uint64_t touched;
  uint64_t input_bound_violations;
  double direction_seconds;
  double label_seconds;
} mssz_oracle_stats;

const char* mssz_oracle_last_error(void);
void mssz_oracle_free(void* p);
int mssz_oracle_build_topology(int ndims, const uint64_t* dims, uint64_t* vertex_count);
int mssz_oracle_neighbors(int ndims, const uint64_t* dims, uint64_t v, uint64_t* out, int* n);
int mssz_oracle_compute_labels(int ndims, const uint64_t* dims, const uint64_t* asc,
                               const uint64_t* desc, uint64_t* max_label, uint64_t* min_label);

#define MSSZ_ORACLE_DECLARE(SUF, T)                                                          \
  int mssz_oracle_compute_directions_##SUF(int ndims, const uint64_t* dims, const T* values,  \
                                           uint64_t* asc, uint64_t* desc);                   \
  int mssz_oracle_detect_false_critical_##SUF(int ndims, const uint64_t* dims, const T* f,    \
                                              const T* g, uint64_t* counts, uint64_t* lists); \
  int mssz_oracle_detect_kind_##SUF(int ndims, const uint64_t* dims, const T* f, const T* g,  \
                                    int kind, uint64_t* list, uint64_t* count);               \
  T mssz_oracle_representable_floor_##SUF(T f, double xi);                                    \
  int mssz_oracle_lower_step_##SUF(T* g, T f, double xi);                                     \
  int mssz_oracle_derive_edits_##SUF(int ndims, const uint64_t* dims, const T* f,             \
                                     const T* fhat, double xi, const mssz_oracle_options* o,  \
                                     void (*on_batch)(const T*, uint64_t, void*), void* user, \
                                     uint64_t** idx, T** val, uint64_t* count,                \
                                     mssz_oracle_stats* stats);

MSSZ_ORACLE_DECLARE(f32, float)
MSSZ_ORACLE_DECLARE(f64, double)

#ifdef __cplusplus
}
#endif
#endif
