/* qswg — B200-native Lindblad expmv for quantum stochastic walks: C ABI.
 *
 * The drop-in boundary for the reference's hot path.  The
 * reference (/root/reference/proj, C++20) exposes no plugin/FFI layer; its
 * boundary is the C++ library surface below, and every entry point here names
 * the reference declaration it replaces (paths under proj/core/include/qsw/).
 * INTEGRATION.md shows the ctypes / C++ bindings a maintainer would add.
 *
 * Conventions
 *  - Complex values are interleaved (re, im) doubles; indices are int64.
 *  - vec(rho) is column-major: element k = n*j + i holds rho(i, j)
 *    (state.hpp:10-12).
 *  - Host arrays passed in are borrowed for the duration of the call.
 *  - Handles own device memory; they are not thread-safe per handle.
 *  - Every function returns QSWG_OK or an error code; qswg_last_error()
 *    returns the thread-local message.  No exception crosses the ABI.
 *  - There is no CPU fallback: without a CUDA device the device entry points
 *    fail with QSWG_ECUDA.
 */
#ifndef QSWG_H
#define QSWG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSWG_VERSION_MAJOR 0
#define QSWG_VERSION_MINOR 1

enum {
  QSWG_OK = 0,
  QSWG_EINVAL = 1,     /* std::invalid_argument  */
  QSWG_ERANGE = 2,     /* std::out_of_range      */
  QSWG_ENUMERICAL = 3, /* qsw::NumericalError    */
  QSWG_ESTATE = 4,     /* std::logic_error       */
  QSWG_ECUDA = 5,
  QSWG_ENCCL = 6,
  QSWG_ENOMEM = 7,
  QSWG_EINTERNAL = 9,
  QSWG_EFORMAT = 10,   /* qsw::FileFormatError (graph.hpp:11-15) */
  QSWG_EIO = 11        /* qsw::IoError (container.hpp:13-17)      */
};

typedef struct qswg_sparse qswg_sparse;           /* host canonical CSR, complex128 */
typedef struct qswg_liouvillian qswg_liouvillian; /* device superoperator (row block) */
typedef struct qswg_state qswg_state;             /* device vec(rho) (row block)     */
typedef struct qswg_comm qswg_comm;               /* multi-GPU communicator          */
typedef struct qswg_container qswg_container;     /* host QSWBOX result container    */

typedef struct { int64_t target; double rate; } qswg_source_arc; /* graph.hpp:17-20 SourceArc */
typedef struct { int64_t origin; double rate; } qswg_sink_arc;   /* graph.hpp:23-26 SinkArc   */

enum { QSWG_FORMAT_AUTO = 0, QSWG_FORMAT_CSR = 1, QSWG_FORMAT_SELL = 2, QSWG_FORMAT_KRON = 3 };

typedef struct {
  int device;       /* CUDA ordinal */
  int group;        /* CSR lanes per row (2..32); 1 = bitwise reference order; 0 = autotune */
  int format;       /* QSWG_FORMAT_*: how the superoperator is applied.  KRON: matrix-free
                       action on the n x n operators, nothing N^2 x N^2 stored; SELL: stored
                       sliced-ELL (32-row slices); CSR: stored CSR.  AUTO = KRON, except in
                       the bitwise mode (group = 1), where it is SELL if its padding is
                       <= 3 %, else CSR. */
  qswg_comm* comm;  /* NULL for one GPU */
} qswg_device_config;

typedef struct {
  int64_t n, dim, nnz, nnz_local, row0, rows;
  double omega;
  double one_norms[9]; /* DistributedLiouvillian::one_norms(), liouvillian.hpp:31 */
  int group, device, rank, world;
  int format;     /* QSWG_FORMAT_CSR, QSWG_FORMAT_SELL or QSWG_FORMAT_KRON */
  double padding; /* stored entries / nnz_local */
  int kron_factored; /* KRON: G-QSW L'L terms applied in factored form */
  int kron_ell;      /* KRON: row-indexed operands read in sliced ELL */
  int kron_term_vectors; /* KRON: n^2 work vectors per Lindblad term the (Hermitian-path) term
                            kernel reads and the prepare kernel writes (roofline bytes) */
  int sell_panels;    /* SELL: column panels of the stored superoperator (1 = one pass; 0 other formats) */
  int kron_hermitian; /* KRON: the last product / step / series ran the Hermitian tile kernels */
  int kron_staged;    /* KRON: the Hermitian series term stages its operand tiles in shared memory
                         (opt-in; lattice-like operands, n a multiple of 32, one GPU) */
  int sell_fused;     /* SELL: the B (x) I entries are kept in natural row order beside the sorted rest
                         (coalesced gathers; one GPU, sigma-sorted superoperators) */
} qswg_liouvillian_info;

typedef struct { int64_t m_star, s, spmvs, launches; } qswg_step_info;

typedef struct {
  int path; /* 0 zero generator, 1 sequential steps, 2 shared-term super-steps */
  int64_t span_m_star, span_s, d, n_super, remainder, sub_m_star, spmvs;
  int64_t launches; /* qswg kernels enqueued by the call */
  double device_ms; /* CUDA-event time of the whole series on the library stream */
  int64_t host_waits; /* several GPUs: host waits for a stop flag (bounded run-ahead); the
                         stream is synchronised once per call, never per term */
} qswg_series_info;

const char* qswg_last_error(void);
int qswg_version(int* major, int* minor);
int qswg_device_count(int* count);
/* Page-locked host buffers (cudaHostAlloc / cudaFreeHost): uploads from and
 * population reads into them are DMA transfers without a staging copy.  No
 * reference counterpart (host vectors are std::vector there). */
int qswg_host_alloc(int64_t bytes, void** out);
void qswg_host_free(void* p);

/* ---- host sparse matrices (sparse.hpp:29-84) ---------------------------- */
/* SparseMatrix::from_triplets (sparse.hpp:35-37): sort, sum duplicates, drop zeros. */
int qswg_sparse_from_triplets(int64_t rows, int64_t cols, int64_t count, const int64_t* row,
                              const int64_t* col, const double* val, qswg_sparse** out);
/* Canonicalising import of CSR arrays. */
int qswg_sparse_from_csr(int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* col,
                         const double* val, qswg_sparse** out);
int qswg_sparse_shape(const qswg_sparse* m, int64_t* rows, int64_t* cols, int64_t* nnz);
int qswg_sparse_export(const qswg_sparse* m, int64_t* rowptr, int64_t* col, double* val);
void qswg_sparse_destroy(qswg_sparse* m);

/* ---- graph -> operators (graph.hpp:78-96, operators.hpp:53-57) ---------- */
int qswg_symmetrize(const qswg_sparse* adjacency, qswg_sparse** out);
int qswg_generator_matrix(double gamma, const qswg_sparse* adjacency, qswg_sparse** out);
int qswg_markov_chain_matrix(const qswg_sparse* adjacency, qswg_sparse** out);
int qswg_local_lindblad(const qswg_sparse* m, qswg_sparse** out);
int qswg_augment(const qswg_sparse* adjacency, const qswg_source_arc* sources, int64_t n_sources,
                 const qswg_sink_arc* sinks, int64_t n_sinks, qswg_sparse** out);

/* ---- non-moralising G-QSW operators (operators.hpp:16-83) --------------- */
/* nm_vsets(gu): dims[i] = arcs into vertex i of the symmetric gu, at least 1. */
int qswg_nm_vsets(const qswg_sparse* gu, int64_t* dims);
/* nm_H(gamma, gu, V), nm_L(gamma, g, V), nm_H_rot(V, dim2) for V given by dims[n_vertices]. */
int qswg_nm_H(double gamma, const qswg_sparse* gu, const int64_t* dims, int64_t n_vertices, qswg_sparse** out);
int qswg_nm_L(double gamma, const qswg_sparse* g, const int64_t* dims, int64_t n_vertices, qswg_sparse** out);
int qswg_nm_H_rot(const int64_t* dims, int64_t n_vertices, int pauli_y, qswg_sparse** out);
/* nm_rho_map(p, V) -> expanded[sum(dims)]; nm_measure(diag, V) -> p[n_vertices]. */
int qswg_nm_rho_map(const double* p, const int64_t* dims, int64_t n_vertices, double* expanded);
int qswg_nm_measure(const double* diag, const int64_t* dims, int64_t n_vertices, double* p);

/* ---- superoperator (liouvillian.hpp:65-93) ------------------------------ */
/* build_local(omega, h, m_l, sources, sinks, n_workers), liouvillian.hpp:65-71 */
int qswg_build_local(double omega, const qswg_sparse* h, const qswg_sparse* m_l,
                     const qswg_source_arc* sources, int64_t n_sources, const qswg_sink_arc* sinks,
                     int64_t n_sinks, const qswg_device_config* cfg, qswg_liouvillian** out);
/* build_global(omega, h, lindblads, h_rot, n_workers), liouvillian.hpp:73-85 */
int qswg_build_global(double omega, const qswg_sparse* h, const qswg_sparse* const* lindblads,
                      int64_t n_lindblads, const qswg_sparse* h_rot /* nullable */,
                      const qswg_device_config* cfg, qswg_liouvillian** out);
int qswg_liouvillian_query(const qswg_liouvillian* l, qswg_liouvillian_info* info);
/* KRON on one GPU: 1 (default) lets step/series/spmv take the Hermitian tile
 * kernels when their input is exactly Hermitian, 0 always uses the general
 * kernels (results agree to rounding; no reference counterpart). */
int qswg_liouvillian_set_hermitian_mode(qswg_liouvillian* l, int mode);
/* gather_full() of the local row block (liouvillian.hpp:34): rowptr[rows+1], col[nnz_local], val[2*nnz_local] */
/* WalkSystem::set_omega (walk.hpp:58, walk.cpp:141-145) on the built operator:
 * re-mixes the superoperator for a new omega in place on the device (same
 * handle, same row partition; states of this handle stay valid), with the
 * 1-norm series recomputed.  EINVAL unless 0 <= omega <= 1. */
int qswg_liouvillian_set_omega(qswg_liouvillian* l, double omega);
int qswg_liouvillian_download(const qswg_liouvillian* l, int64_t* rowptr, int64_t* col, double* val);
void qswg_liouvillian_destroy(qswg_liouvillian* l);
/* spmv(l, x), liouvillian.hpp:93: y = L x; x: dim complex (host), y: rows complex (host) */
int qswg_spmv(const qswg_liouvillian* l, const double* x, double* y);
/* Mean device time of one plain SpMV kernel over `iters` back-to-back launches. */
int qswg_time_spmv(const qswg_liouvillian* l, int iters, int group, double* ms);
/* Mean device time of one series term (Kron prepare + term kernel + the
 * amortised running-sum flush of `count` outputs) over `iters` terms. */
int qswg_time_series_term(const qswg_liouvillian* l, int iters, int count, double* ms);
/* The same split into its parts: ms4 = {prepare, term kernel, flush, total}. */
int qswg_time_series_parts(const qswg_liouvillian* l, int iters, int count, double* ms4);
/* The CUDA stream (cudaStream_t) every kernel of this handle runs on. */
int qswg_liouvillian_stream(const qswg_liouvillian* l, void** stream);

/* ---- states (state.hpp:13-27, walk.hpp:57-66) --------------------------- */
int qswg_state_create(const qswg_liouvillian* l, qswg_state** out);
/* StateVector::scatter(full) — uploads this rank's rows of a full host vec(rho).
 * On one GPU (matrix-free format) the state's exact Hermiticity is checked on
 * the device here, once, so later step/series calls on it do not synchronise
 * for it. */
int qswg_state_upload(qswg_state* s, const double* vec);
/* WalkSystem::initial_state(probabilities) (walk.cpp:101-126), built on the device */
int qswg_state_from_probabilities(qswg_state* s, const double* p, int64_t n);
/* StateVector::gather() of this rank's rows */
int qswg_state_download(const qswg_state* s, double* vec);
/* populations_of(state) (walk.cpp:177-186): out[n] (zeros for diagonals owned by other ranks) */
int qswg_state_populations(const qswg_state* s, double* out);
void qswg_state_destroy(qswg_state* s);

/* ---- Taylor parameters (expm.hpp:19-45) --------------------------------- */
int qswg_theta_table(double tolerance, double* theta55);
int qswg_select_parameters(const double* one_norms9, double t, double tolerance, int64_t* m_star,
                           int64_t* s);

/* ---- evolution (expm.hpp:47-63) ----------------------------------------- */
/* out = exp(t L) v  (qsw::step). out must be a distinct state of the same L. */
int qswg_step(const qswg_liouvillian* l, const qswg_state* v, double t, double tolerance,
              qswg_state* out, qswg_step_info* info);
/* qsw::series over [t1, tq] with `steps` intervals.  pops_host: (steps+1)*n
 * doubles or NULL (populations then stay on the device); states_host:
 * (steps+1)*rows complex or NULL; final_state: receives the tq state or NULL. */
int qswg_series(const qswg_liouvillian* l, const qswg_state* v, double t1, double tq, int64_t steps,
                double tolerance, double* pops_host, double* states_host, qswg_state* final_state,
                qswg_series_info* info);

/* qswg_series plus the coherence norm of every output state, computed on the
 * device: coherence_host[(steps+1)] = max_{i != j} |rho_k(i, j)|, what
 * run() stores as "coherence_norm" from DensityMatrix::max_coherence of each
 * gathered state (run.cpp:124-137, walk.cpp:32-40).  NULL skips it. */
int qswg_series_observe(const qswg_liouvillian* l, const qswg_state* v, double t1, double tq, int64_t steps,
                        double tolerance, double* pops_host, double* coherence_host, double* states_host,
                        qswg_state* final_state, qswg_series_info* info);
/* max_{i != j} |rho(i, j)| of one state (DensityMatrix::max_coherence, walk.hpp:25). */
int qswg_state_coherence(const qswg_state* s, double* out);

/* ---- file formats either side of the path ------ */
/* WeightedDigraph::load_matrix_market (graph.cpp:54-136) on an in-memory
 * stream: the adjacency matrix (entry (i, j) = arc j -> i).  Format errors
 * -> QSWG_EFORMAT; self-loops / non-positive weights -> QSWG_EINVAL. */
int qswg_matrix_market_parse(const char* text, int64_t len, qswg_sparse** adjacency);
/* The graph-file loader of run() (run.cpp:14-25): QSWG_EIO when the file
 * cannot be opened, every other failure QSWG_EFORMAT naming the file. */
int qswg_matrix_market_load(const char* path, qswg_sparse** adjacency);
/* WeightedDigraph::save_matrix_market (graph.cpp:138-150). */
int qswg_matrix_market_save(const qswg_sparse* adjacency, const char* path);
/* ResultContainer (container.hpp:19-46): metadata text + named float64
 * arrays (row-major, explicit shape), QSWBOX v1 bytes on disk. */
int qswg_container_create(qswg_container** out);
void qswg_container_destroy(qswg_container* c);
int qswg_container_set_metadata(qswg_container* c, const char* text, int64_t len);
int qswg_container_get_metadata(const qswg_container* c, char* buf, int64_t cap, int64_t* len);
/* Inserts or replaces array `name`; data holds prod(shape) doubles. */
int qswg_container_put_array(qswg_container* c, const char* name, int64_t rank, const int64_t* shape,
                             const double* data);
int qswg_container_array_count(const qswg_container* c, int64_t* count);
/* Arrays are enumerated in name order (the on-disk order). */
int qswg_container_array_info(const qswg_container* c, int64_t index, char* name, int64_t name_cap,
                              int64_t* name_len, int64_t* rank, int64_t* shape, int64_t shape_cap);
int qswg_container_array_data(const qswg_container* c, int64_t index, double* data);
/* write_container / read_container (container.hpp:48-49). */
int qswg_container_write(const qswg_container* c, const char* path);
int qswg_container_read(const char* path, qswg_container** out);
/* emit_plot_data (container.hpp:51-56) into a text file. */
int qswg_container_plot_data(const qswg_container* c, const char* quantity, const char* path);

/* ---- multi-GPU (one process per GPU) ------------------------------------ */
/* Row partition on rho-column boundaries balanced by nnz (the device build
 * uses the same function; replaces RowPartition::even, partition.cpp:8-19):
 * colptr[j] = nnz before rho column j (n+1 entries) -> starts[world+1]. */
int qswg_plan_rows(int64_t n, const int64_t* colptr, int world, int64_t* starts);
/* Halo plan of one rank (replaces plan_communication, partition.cpp:26-59):
 * hull [lo[q], hi[q]) of the columns in cols[] owned by peer q (empty: lo == hi). */
int qswg_plan_halo(const int64_t* cols, int64_t nnz, const int64_t* starts, int world, int rank, int64_t* lo,
                   int64_t* hi);
/* The partition (starts[world+1]) and halo table (world x world, row r =
 * what rank r receives from each peer) of a built superoperator. */
int qswg_liouvillian_partition(const qswg_liouvillian* l, int64_t* starts, int64_t* halo_lo, int64_t* halo_hi);
int qswg_comm_unique_id_size(void);
int qswg_comm_get_unique_id(uint8_t* id);
int qswg_comm_create(const uint8_t* id, int rank, int world, int device, qswg_comm** out);
void qswg_comm_destroy(qswg_comm* c);
/* `world` linked in-process communicators, one per host thread: runs the
 * multi-GPU control flow (halo exchanges, allreduces) inside one process,
 * e.g. several ranks on one GPU for testing; collectives are host-side
 * rendezvous, so no kernel waits on another rank. */
int qswg_comm_create_local(int world, qswg_comm** outs);

#ifdef __cplusplus
}
#endif
#endif /* QSWG_H */
