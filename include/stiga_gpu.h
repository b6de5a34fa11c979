/*
 * stiga_gpu.h -- C ABI of the B200-native extended-FD preconditioner / GMRES hot path.
 *
 * This is the drop-in boundary for the reference's C++ operator/solver API
 * (/root/reference/proj/core/include/stiga/ headers).  Every entry point names the reference
 * interface it replaces.  Plain pointers and sizes only; no C++ or torch types.
 *
 * Conventions (mirroring the reference):
 *   - FP64 everywhere; vectors are colexicographic (i_1 fastest, time slowest), kronop.hpp:10-13.
 *   - Dense matrices are column-major n x n (the reference's BandedMatrix stores dense, assembly.hpp:18-36).
 *   - Every call returns a status: STIGA_OK, STIGA_INVALID_ARGUMENT (std::invalid_argument in the
 *     reference), STIGA_NUMERICAL (std::runtime_error), STIGA_CUDA (device failure).
 *     stiga_last_error() returns the message of the last failure on the calling thread.
 *   - Handles are immutable after setup; apply is reentrant per (handle, stream) pair when the
 *     caller passes distinct output buffers (scratch is per handle: concurrent applies on one
 *     handle from several streams are not allowed).
 *   - "device" pointers are CUDA global-memory pointers on the handle's device; "host" pointers
 *     are ordinary host memory (pinned or pageable).
 */
#ifndef STIGA_GPU_H
#define STIGA_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

#define STIGA_OK 0
#define STIGA_INVALID_ARGUMENT 1
#define STIGA_NUMERICAL 2
#define STIGA_CUDA 3

typedef struct stiga_fd_s* stiga_fd_t;
typedef struct stiga_kronsum_s* stiga_kronsum_t;
typedef struct stiga_problem_s* stiga_problem_t;

/* ---- diagnostics ------------------------------------------------------------------- */

/* Message of the last failed call on this thread ("" if none). */
const char* stiga_last_error(void);
/* ABI version (major*100 + minor). */
int stiga_abi_version(void);
/* Number of CUDA devices visible (0 on a machine without GPU); never fails. */
int stiga_device_count(void);

/* ---- host-side 1D assembly (stays on the host, as in the reference) ------------------ */

/* Active dimension of SplineSpace1D::spatial (kind 0) / ::temporal (kind 1), bspline.cpp:139-145. */
int stiga_space_dim(int p, int n_el, int kind, int* n_out);
/* assemble_time_matrices(p_t, n_el_t, T) -> W_t, M_t (assembly.cpp:129-138); Wt, Mt are n_t*n_t. */
int stiga_assemble_time_matrices(int p_t, int n_el_t, double T, double* Wt, double* Mt);
/* assemble_spatial_parametric for one direction with q Gauss points per element
   (assembly.cpp:140-149): K, M are n_s*n_s. */
int stiga_assemble_spatial_parametric(int p, int n_el, int q, double* K, double* M);
/* assemble_univariate with per-element weights (assembly.cpp:47-79, overload 118-127);
   kind 0 = spatial space, 1 = temporal space; weights may be NULL (all ones). out: n*n. */
int stiga_assemble_univariate(int p, int n_el, int kind, int q, int deriv_row, int deriv_col,
                              const double* element_weights, double* out);

/* ---- problems, geometry and the A^G coefficient pieces (host) -------------------------- */

/* make_problem(id) (problems.cpp:244-261), geometry + coefficient part: "identity-interval-1d",
   "identity-square-2d", "identity-cube-3d", "quarter-annulus-2d", "separable-nu-2d", and the
   BASELINE config-4 "deformed-cube-3d" (fit_geometry of x + 0.1 sin sin sin (1,1,1) with p_g=3,
   n_el_g=8; kappa = 1 + 0.5 sin(2 pi x1) cos(2 pi x2); c = 1 + 0.25 x3). */
int stiga_problem_create(const char* id, stiga_problem_t* out);
int stiga_problem_destroy(stiga_problem_t P);
int stiga_problem_dim(stiga_problem_t P, int* d);
/* GeometryMap::value / ::jacobian (geometry.cpp:41-97); J is column-major d x d, x or J may be NULL. */
int stiga_problem_eval_geometry(stiga_problem_t P, const double* eta, double* x, double* J);
/* nu_s(x), gamma_s(x) of the problem (1 when constant). */
int stiga_problem_eval_fields(stiga_problem_t P, const double* x, double* nu_s, double* gamma_s);
/* Inputs of make_geometry_preconditioner (solver.cpp:127-144) for degree p / n_el elements in every
   direction and in time: K~_l, M~_l (d blocks of n_s*n_s, column-major), W_t and the weighted M_t
   (n_t*n_t), D = diag(A)/diag(A~) (N_dof; NULL skips the physical diagonal quadrature), the separated
   factors phi, Phi (d*n_el each, may be NULL), the fit residuals (d+1) and ALS sweeps (may be NULL). */
int stiga_geometry_preconditioner_pieces(stiga_problem_t P, int p, int n_el, double* Kt, double* Mt_s, double* Wt,
                                         double* Mt, double* D, double* phi, double* Phi, double* residuals,
                                         int* sweeps);

/* ---- ExtendedFDPreconditioner (fdsolve.hpp:41-70) ------------------------------------- */

/* ExtendedFDPreconditioner::setup(space_K, space_M, Wt, Mt, gamma, nu, scaling) (fdsolve.hpp:48-52,
   fdsolve.cpp:67-153).  d directions; K[l], M[l] point to n[l]*n[l] column-major matrices;
   Wt, Mt are n_t*n_t.  scaling (the optional D, length scaling_len == N_dof) may be NULL.
   The eigen/pencil factorizations run on the host; factors are uploaded to `device` once. */
int stiga_fd_setup(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                   const double* Wt, const double* Mt, double gamma, double nu, const double* scaling,
                   long long scaling_len, int device, stiga_fd_t* out);
/* device < 0 creates a host-only handle (setup + stiga_fd_export, no device apply). */

/* Device-side setup.  STIGA_SETUP_DEVICE_SCHUR: Lambda_s and the Schur diagonal S^-1
   (fdsolve.cpp:91-136) computed on the device, bit-identical to the host loop (correctly rounded
   arithmetic in the host's operation order); STIGA_SETUP_CUSOLVER: every symmetric eigenproblem of the
   setup (spatial pencils after the Cholesky reduction, the split half-pencils, the Hermitian embedding of
   the time pencil) solved by cuSOLVER syevd on `device`.  d_scaling: D (scaling_len == N_dof entries) in
   DEVICE memory instead of the host `scaling`; D^-1/2 is then formed on the device (unsharded handles). */
#define STIGA_SETUP_DEVICE_SCHUR 1
#define STIGA_SETUP_CUSOLVER 2
typedef struct {
    int flags;
    const double* d_scaling;
} stiga_fd_setup_options;
int stiga_fd_setup_ex(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                      const double* Wt, const double* Mt, double gamma, double nu, const double* scaling,
                      long long scaling_len, const stiga_fd_setup_options* opts, int device, stiga_fd_t* out);
int stiga_fd_destroy(stiga_fd_t P);
/* ExtendedFDPreconditioner::size() and the tensor dims (d spatial sizes then n_t). */
int stiga_fd_size(stiga_fd_t P, long long* n_dof);
int stiga_fd_dims(stiga_fd_t P, int* d, int* dims);
/* Time-factorization summary: #pairs, zero_count, sigma, rho (pencil.hpp:40-52). */
int stiga_fd_time_info(stiga_fd_t P, int* npairs, int* zero_count, double* sigma, double* rho);
/* Copies host-side factors for inspection: which = 0: U_l (n_l*n_l, col-major) for direction l;
   1: Lambda_l (n_l); 2: U_t (n_t*n_t); 3: lambda_t (npairs); 4: g (n_t-1); 5: S_inv (N_s). */
int stiga_fd_export(stiga_fd_t P, int which, int l, double* out, long long out_len);

/* ExtendedFDPreconditioner::apply(r) (fdsolve.hpp:56, fdsolve.cpp:155-164) on device buffers,
   asynchronously on `stream` (a cudaStream_t, NULL = legacy default stream).  d_s may equal d_r. */
int stiga_fd_apply(stiga_fd_t P, const double* d_r, double* d_s, void* stream);
/* Host-buffer convenience: H2D copy, apply, D2H copy, synchronize. */
int stiga_fd_apply_host(stiga_fd_t P, const double* h_r, double* h_s);
/* Same as stiga_fd_apply but records CUDA events around each of the kernel launches (2d+1, +1 post-scale with D) and
   writes their durations (ms) into pass_ms[0..launches-1] (synchronizes the stream). */
int stiga_fd_apply_profiled(stiga_fd_t P, const double* d_r, double* d_s, void* stream, float* pass_ms);
/* Number of kernel launches one apply issues (2d+1, +1 when scaled by D). */
int stiga_fd_launches(stiga_fd_t P, int* launches);
/* Name (e.g. "fwd_mode0", "time_fused", "arrowhead") and algorithmic FP64 flops of launch i of an
   apply (the dense mode-product flops 2 n N_dof per product; 0 for elementwise passes). */
int stiga_fd_launch_info(stiga_fd_t P, int i, char* name, int name_len, double* flops);

/* ---- distributed (time-sharded) apply building blocks, DESIGN.md §6 ------------------------ */

/* Spatial half of the apply on a time slab (time slices [t0, t0+nt_local), a contiguous piece of
   the colex vector): forward = D^-1/2 pre-scale of the slab (when scaled) + U_1^T..U_d^T;
   backward = U_1..U_d with the D^-1/2 post-scale fused.  d_in != d_out. */
int stiga_fd_apply_space(stiga_fd_t P, int backward, long long t0, long long nt_local, const double* d_in,
                         double* d_out, void* stream);
/* Time direction (U_t^T, arrowhead_solve fdsolve.cpp:24-65, U_t) on a spatial slab: ns_local spatial
   eigen-indices starting at global index s0, stored ns_local x n_t colexicographically. */
int stiga_fd_apply_time(stiga_fd_t P, long long s0, long long ns_local, const double* d_in, double* d_out,
                        void* stream);
/* Fused exchange: the same two stages, but the last product of the stage stores every
   output element straight into the receive buffer of the rank that owns it -- the all-to-all
   transpose of the time-sharded apply fused into the producing kernel's epilogue (NVLink P2P stores
   through pointers opened with stiga_ipc_open; plain local pointers for virtual ranks).  Replaces
   pack + all-to-all + unpack; the caller orders the stages across ranks (a barrier after each
   scatter stage).  Destination of output element (a, b):
     dst[q] + (a - (by_time ? 0 : offsets[q]) + a_shift) + ld[q] * (b - (by_time ? offsets[q] : 0) + b_shift)
   space stage (by_time = 0): a = spatial index (0..N_s), b = local time slice; q owns a;
   time stage  (by_time = 1): a = local spatial index (0..ns_local), b = time slice; q owns b.
   offsets[0..world] partition the owner coordinate (increasing, offsets[world] = its extent). */
#define STIGA_MAX_RANKS 8
#define STIGA_IPC_HANDLE_BYTES 64
typedef struct stiga_scatter_desc {
    int world;
    int by_time;
    long long offsets[STIGA_MAX_RANKS + 1];
    long long ld[STIGA_MAX_RANKS];
    long long a_shift, b_shift;
    double* dst[STIGA_MAX_RANKS];
} stiga_scatter_desc;
/* Forward spatial stage (pre-scale + U_1^T..U_d^T) of time slab [t0, t0+nt_local), scattered. */
int stiga_fd_apply_space_scatter(stiga_fd_t P, long long t0, long long nt_local, const double* d_in,
                                 const stiga_scatter_desc* sc, void* stream);
/* Time stage (U_t^T, arrowhead, U_t) of spatial slab [s0, s0+ns_local), scattered. */
int stiga_fd_apply_time_scatter(stiga_fd_t P, long long s0, long long ns_local, const double* d_in,
                                const stiga_scatter_desc* sc, void* stream);
/* Plain cudaMalloc / cudaFree on `device` (receive buffers that can be shared with CUDA IPC). */
int stiga_device_alloc(long long bytes, int device, void** d_ptr);
int stiga_device_free(void* d_ptr);
/* CUDA IPC: export a cudaMalloc'd base pointer (STIGA_IPC_HANDLE_BYTES opaque bytes), open a peer's
   handle in this process (peer access enabled lazily), close it. */
int stiga_ipc_handle(const void* d_ptr, void* handle_out);
int stiga_ipc_open(const void* handle, int device, void** d_ptr);
int stiga_ipc_close(void* d_ptr);

/* Strided block copy dst[r*dst_ld + c] = src[r*src_ld + c] (pack/unpack around the all-to-alls). */
int stiga_copy_blocks(const double* d_src, long long src_ld, double* d_dst, long long dst_ld, long long rows,
                      long long cols, void* stream);

/* ---- multi-GPU: communicator and time-sharded handles ------------------------
   One process per GPU.  Rank r owns the time slices T_r = [t_off[r], t_off[r] + t_len[r]) of every
   N_dof vector (a contiguous piece of the colex vector; balanced contiguous partition of n_t, the
   first n_t % world ranks get one slice more -- stiga_shard_partition).  A sharded handle's apply,
   mat-vec and GMRES take and return only the local slab; every rank calls them collectively.
   The reference is serial; this is new work, not a replacement of a reference API. */
typedef struct stiga_comm_s* stiga_comm_t;
#define STIGA_COMM_ID_BYTES 128
/* NCCL unique id (ncclGetUniqueId) for rank 0 to broadcast out of band. */
int stiga_comm_unique_id(void* id_out);
/* NCCL communicator of this rank over `world` ranks (ncclCommInitRank; NCCL is loaded at run time).
   Collectives and barriers are stream-ordered on the caller's stream. */
int stiga_comm_init_nccl(int world, int rank, const void* id, int device, stiga_comm_t* out);
/* Host-callback communicator: the caller supplies the collectives (e.g. over an existing process
   group); the library synchronizes the stream before calling them.  allreduce reduces n host doubles
   in place (op 0 = sum, 1 = max); allgather gathers `bytes` from every rank into recv (world x bytes,
   rank order).  Each returns 0 on success. */
typedef struct {
    void* ctx;
    int (*allreduce)(void* ctx, double* buf, int n, int op);
    int (*allgather)(void* ctx, const void* send, int bytes, void* recv);
    int (*barrier)(void* ctx);
} stiga_comm_callbacks;
int stiga_comm_init_host(int world, int rank, const stiga_comm_callbacks* cb, int device, stiga_comm_t* out);
int stiga_comm_destroy(stiga_comm_t C);
/* world, rank, device, kind (0 = NCCL, 1 = host callbacks); any output may be NULL. */
int stiga_comm_info(stiga_comm_t C, int* world, int* rank, int* device, int* kind);
/* Sum-all-reduce of n doubles of device memory (stream-ordered for NCCL). */
int stiga_comm_allreduce(stiga_comm_t C, double* d_buf, long long n, void* stream);
/* Balanced contiguous partition of range(n) over world parts: offset and length of part `rank`. */
int stiga_shard_partition(long long n, int world, int rank, long long* off, long long* len);

/* Time-sharded ExtendedFDPreconditioner (collective): the same host setup on every rank, then the
   rank's stage kernels are tuned on its slab geometry.  scaling_local: D for the local time slab only
   (N_s x t_len[rank] entries, colex), or NULL.  Device memory per rank ~ 4-5 N_dof / world doubles
   (two scratch slabs, two receive buffers, the D^-1/2 slab) plus the factors.  stiga_fd_apply on
   the handle then runs the sharded apply on local slabs: forward spatial products with the last one
   scattering into the owners' spatial-slab buffers (the all-to-all fused into the epilogue, NVLink P2P
   stores through CUDA IPC pointers), a stream-ordered barrier, the time stage (U_t^T, arrowhead, U_t)
   on the rank's spatial slab scattering back into the owners' time-slab buffers, a barrier, and the
   backward spatial products with the D^-1/2 post-scale. */
int stiga_fd_setup_sharded(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                           const double* Wt, const double* Mt, double gamma, double nu, const double* scaling_local,
                           long long scaling_len, stiga_comm_t comm, stiga_fd_t* out);
/* Local slab of a handle: time slices [*t0, *t0 + *nt_local), i.e. vector entries [*offset, *offset + *len)
   of the global colex vector (t0 = 0, nt_local = n_t for a single-device handle). */
int stiga_fd_local(stiga_fd_t P, long long* t0, long long* nt_local, long long* offset, long long* len);

/* ---- Kronecker operators (kronop.hpp:47-79) ------------------------------------------- */

/* kron_matvec(factors, x) (kronop.cpp:75-89) on device buffers: D factors, factor l is
   rows[l] x cols[l] column-major (host pointer); x has prod(cols) entries, y prod(rows). */
int stiga_kron_matvec(int D, const int* rows, const int* cols, const double* const* factors,
                      const double* d_x, double* d_y, int device, void* stream);

/* KronSumOperator(dims, terms) (kronop.hpp:61-79): D dims, nterms terms; term t has coefficient
   coeffs[t] and D square factors factors[t*D + l] (dims[l]^2, column-major, host pointers).
   Banded factors are detected and applied with banded kernels. */
int stiga_kronsum_create(int D, const int* dims, int nterms, const double* coeffs,
                         const double* const* factors, int device, stiga_kronsum_t* out);
/* KronSumOperator(dims, kron_sum_terms(K, M, Wt, Mt, gamma, nu)) (solver.cpp:10-30, 67-70): the
   (d+1)-term space-time operator  gamma (M_1..M_d, W_t) + nu sum_l (M_1..K_l..M_d, M_t)  with
   banded 1D factors, applied sum-factorized in d+1 banded passes (equal to the per-term sum in
   exact arithmetic).  K[l], M[l]: n[l]*n[l]; Wt, Mt: n_t*n_t (column-major, host pointers). */
int stiga_kronsum_create_spacetime(int d, const int* n, const double* const* K, const double* const* M,
                                   int n_t, const double* Wt, const double* Mt, double gamma, double nu,
                                   int device, stiga_kronsum_t* out);
/* SpaceTimeSystem's A_ = M_s (x) W_t + K_s (x) M_t (solver.cpp:58-70) with the physical spatial
   matrices of `prob` (assemble_spatial_physical, assembly.cpp:151-268) assembled on the device
   (one CTA per element, stencil storage of the (2p+1)^d tensor B-spline neighbours) for degree p,
   n_el elements per direction and in time; the time mass carries nu_t/gamma_t. */
int stiga_kronsum_create_physical(stiga_problem_t prob, int p, int n_el, int device, stiga_kronsum_t* out);
int stiga_kronsum_destroy(stiga_kronsum_t A);
int stiga_kronsum_size(stiga_kronsum_t A, long long* n_dof);
/* Tensor dimensions [n_1 .. n_d, n_t] (*D entries; cap = capacity of dims). */
int stiga_kronsum_dims(stiga_kronsum_t A, int* D, int* dims, int cap);
/* KronSumOperator::apply(x) (kronop.cpp:108-115): y = sum_t coeff_t (x)_l F_{t,l} x. d_y != d_x. */
int stiga_kronsum_apply(stiga_kronsum_t A, const double* d_x, double* d_y, void* stream);
/* KronSumOperator::diagonal() (kronop.cpp:117-131) into a host buffer of N_dof. */
int stiga_kronsum_diagonal(stiga_kronsum_t A, double* h_diag);
/* The same diagonal into a DEVICE buffer of N_dof (bit-identical to stiga_kronsum_diagonal). */
int stiga_kronsum_diagonal_device(stiga_kronsum_t A, double* d_diag, void* stream);
/* make_geometry_preconditioner's D = diag(A) / diag(A~) (solver.cpp:138-142) on the device: A the
   system operator (physical or Kronecker-sum), A~ a Kronecker-sum operator of the same size (the
   separated factors K~, M~, W_t, M_t with gamma = nu = 1).  d_D: N_dof device doubles. */
int stiga_geometry_scaling_device(stiga_kronsum_t A, stiga_kronsum_t Atilde, double* d_D, void* stream);

/* Time-sharded mat-vec building blocks, for the space-time (identity geometry) and
   physical systems: A x = W~ (x) a(x) + M~ (x) b(x) with a, b the spatial halves.
   apply_space: on a slab of nt_local time slices (N_s x nt_local colex), d_a = a(x), d_b = b(x)
     (spacetime: a = (M_d .. M_1) x, b = sum_l (M_d .. K_l .. M_1) x; physical: a = M_s x, b = K_s x).
   apply_time: d_y (slices t0 .. t0+nt_local) = W~ a + M~ b with the time bands (gamma W_t, nu M_t /
     W_t, M_t), where d_a, d_b hold slices [t0 - halo_lo, t0 + nt_local + halo_hi) and each halo is
     min(p, slices that exist) wide (p from stiga_kronsum_time_halfband).  Generic-term operators
     (stiga_kronsum_create) are rejected with STIGA_INVALID. */
int stiga_kronsum_time_halfband(stiga_kronsum_t A, int* p);
int stiga_kronsum_apply_space(stiga_kronsum_t A, long long nt_local, const double* d_x, double* d_a, double* d_b,
                              void* stream);
int stiga_kronsum_apply_time(stiga_kronsum_t A, long long t0, long long nt_local, int halo_lo, int halo_hi,
                             const double* d_a, const double* d_b, double* d_y, void* stream);

/* Time-sharded system operators (collective; same meaning as the single-device constructors below /
   above).  stiga_kronsum_apply then maps the local slab of x to the local slab of y: the spatial halves
   of the slab, a push of the p edge slices into the time neighbours' halos (peer copies through CUDA
   IPC), a stream-ordered barrier, and the banded time pass.  Needs t_len[r] >= p on every rank. */
int stiga_kronsum_create_spacetime_sharded(int d, const int* n, const double* const* K, const double* const* M,
                                           int n_t, const double* Wt, const double* Mt, double gamma, double nu,
                                           stiga_comm_t comm, stiga_kronsum_t* out);
int stiga_kronsum_create_physical_sharded(stiga_problem_t prob, int p, int n_el, stiga_comm_t comm,
                                          stiga_kronsum_t* out);
int stiga_kronsum_local(stiga_kronsum_t A, long long* t0, long long* nt_local, long long* offset, long long* len);

/* GMRES BLAS-1 on the device (gmres.cpp:76-85, 121), for the distributed solver above the ABI:
   deterministic dot into *d_result (device scalar), y += alpha x, y = alpha x. */
int stiga_vec_dot(const double* d_x, const double* d_y, long long n, double* d_result, void* stream);
int stiga_vec_axpy(double alpha, const double* d_x, double* d_y, long long n, void* stream);
/* Batched Krylov operations for classical Gram-Schmidt with reorthogonalisation (CGS2) in the
   sharded GMRES: d_out[j] = V_j . w for j < k (d_V: host array of k <= 64 device pointers, d_out: k
   device doubles, deterministic reduction) and w += sum_j coefs[j] V_j (coefs: k host doubles). */
int stiga_vec_multidot(const double* const* d_V, int k, const double* d_w, long long n, double* d_out, void* stream);
int stiga_vec_multiaxpy(const double* coefs, const double* const* d_V, int k, double* d_w, long long n, void* stream);
int stiga_vec_scal(double alpha, const double* d_x, double* d_y, long long n, void* stream);

/* ---- GMRES (gmres.hpp:12-35) ---------------------------------------------------------- */

/* Mirrors GmresOptions (gmres.hpp:23-27); restart <= 0 means "no restart" (std::nullopt). */
typedef struct {
    double tol;
    int max_krylov;
    int restart;
} stiga_gmres_options;

/* Mirrors SolveReport (gmres.hpp:15-21); residual_history is caller-provided storage of
   history_capacity doubles, history_len receives the number of entries produced. */
typedef struct {
    int iterations;
    int converged;
    double wall_time_s;
    double precond_time_fraction;
    double* residual_history;
    int history_capacity;
    int history_len;
} stiga_gmres_report;

/* gmres(A, P, b, opts) (gmres.cpp:19-132): left-preconditioned GMRES from x0 = 0 with A a
   KronSumOperator handle and P an FD handle (P may be NULL).  d_b, d_x are device buffers.  With
   time-sharded handles (same communicator) d_b, d_x are the local slabs and the solve is collective
   (the CGS2 variant of stiga_gmres_op). */
int stiga_gmres(stiga_kronsum_t A, stiga_fd_t P, const double* d_b, double* d_x,
                const stiga_gmres_options* opts, stiga_gmres_report* report, void* stream);

/* gmres(A, P, b, opts) over caller-supplied operators (gmres.hpp:12 LinOp, gmres.cpp:19-132): A and P
   (P may be NULL) map a device vector of n entries to another on `stream` and return 0 on success.
   With comm != NULL the vectors are this rank's slabs (n local entries) and every Krylov dot is
   all-reduced over the communicator; the Arnoldi column is then orthogonalised by classical
   Gram-Schmidt with one reorthogonalisation (CGS2, two batched reductions per column) instead of the
   reference's MGS (k + 1 sequential reductions).  Without comm the control flow is the reference's MGS. */
typedef int (*stiga_linop_fn)(void* ctx, const double* d_in, double* d_out, void* stream);
int stiga_gmres_op(long long n, stiga_linop_fn A, void* A_ctx, stiga_linop_fn P, void* P_ctx, stiga_comm_t comm,
                   const double* d_b, double* d_x, const stiga_gmres_options* opts, stiga_gmres_report* report,
                   void* stream);

/* ---- space-time system glue (solver.cpp:34-155, assembly.cpp:413-504, problems.cpp:305-402) ---- */

/* ProblemSpec fields (problems.hpp:25-37): d, T, whether the problem carries an analytic source term
   and exact solution (the identity-*, quarter-annulus-2d and separable-nu-2d manufactured problems;
   deformed-cube-3d has none), and the constants gamma0, nu0.  Any output may be NULL. */
int stiga_problem_info(stiga_problem_t P, int* d, double* T, int* has_rhs, int* has_exact, double* gamma0,
                       double* nu0);
/* SpaceTimeSystem's gamma_mean_ / nu_mean_ (solver.cpp:82-112), the constants of
   make_parametric_preconditioner (solver.cpp:122-125); host quadrature with p + 1 Gauss points. */
int stiga_system_means(stiga_problem_t P, int p, int n_el, double* gamma_mean, double* nu_mean);
/* b_ = assemble_rhs(f / gamma_t, T, spatial spaces, time space, geometry, points_per_element)
   (solver.cpp:72-76 with points_per_element = p + 1; assembly.cpp:413-504) into the device vector
   d_b (N_dof, colex, time slowest), sum-factorized on the device.  Returns STIGA_INVALID_ARGUMENT for
   a problem without a source term and STIGA_NUMERICAL for a non-positive Jacobian. Synchronous. */
int stiga_assemble_rhs(stiga_problem_t P, int p, int n_el, int points_per_element, int device, double* d_b,
                       void* stream);
/* compute_errors(u_h, problem, points_per_element) (problems.cpp:305-402) for the device coefficient
   vector d_coeffs (N_dof) of the degree-p / n_el discretisation: relative L2(0,T;L2) error and the
   relative X-norm upper bound.  STIGA_INVALID_ARGUMENT without an exact solution. Synchronous. */
int stiga_compute_errors(stiga_problem_t P, int p, int n_el, const double* d_coeffs, int points_per_element,
                         int device, double* l2l2, double* x_upper);

/* ---- measurement helpers ---------------------------------------------------------------- */

/* Sustained FP64 DMMA (m8n8k4) throughput of the device in TFLOP/s over ~`ms` milliseconds. */
int stiga_fp64_peak(int device, double ms, double* tflops_dmma, double* tflops_dfma);

#ifdef __cplusplus
}
#endif

#endif /* STIGA_GPU_H */
