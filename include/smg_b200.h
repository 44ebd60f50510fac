/* smg_b200.h — C ABI of the B200-native hot path of arXiv 2410.09497 (matrix-free multigrid for the
 * H(div)-DG Stokes problem): Stokes operator vmult, vertex-patch Schur/fast-diagonalisation smoother,
 * intergrid transfer, level vectors, and the V-cycle / mixed-precision FGMRES driver built on them.
 *
 * The reference (/root/reference) ships no code for this path: its interfaces exist as SPEC.md
 * operation signatures plus the BlockVector<dim,T> type (proj/include/stokesmg/block_vector.hpp:15-93).
 * Each entry point below names the reference operation it replaces. Conventions:
 *   - plain pointers and sizes only; no C++ or torch types cross this boundary;
 *   - every call returns an int status (SMG_OK or a negative SMG_E* code); smg_last_error() gives text.
 *     The reference signals errors with std::invalid_argument (mesh.hpp:31-34, fem1d.hpp:95-96);
 *     the C++ wrapper (paper_2410_09497_b200/host/stokesmg_b200.hpp) rethrows them as such;
 *   - device-vector entry points take DEVICE pointers to one contiguous level vector in the stored
 *     layout [u_x | u_y | u_z | p]; *_host entry points take HOST arrays in
 *     the BlockVector layout (3 velocity arrays + pressure, block_vector.hpp:17-18) and copy;
 *   - all device work is ordered on the context's stream (smg_set_stream); calls that return host
 *     scalars (dot, norms, solve) synchronise that stream;
 *   - a context is not re-entrant: one host thread per context.
 * There is no CPU fallback: without a usable sm_100 device smg_create fails with SMG_ECUDA.
 */
#ifndef SMG_B200_H
#define SMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMG_OK 0
#define SMG_EINVAL (-22)   /* std::invalid_argument in the reference */
#define SMG_ECUDA (-100)   /* CUDA runtime / launch failure */
#define SMG_ENOTCONV (-101) /* Krylov did not converge within max_iter */
#define SMG_ENOMEM (-12)

#define SMG_F64 0
#define SMG_F32 1

typedef struct smg_context smg_context;

typedef struct {
  int degree;        /* RT_k velocity / DGQ_k pressure, k >= 1 */
  int max_level;     /* finest level L; level l has 2^(l+1) cells per direction (mesh.hpp:21) */
  int device;        /* CUDA device ordinal */
  int cg_max_iter;   /* patch Schur-CG cap */
  double cg_tol;     /* patch Schur-CG relative tolerance */
  int cg_fixed;      /* 1: exactly cg_max_iter iterations (parity mode) */
  int cg_precond;    /* 0: none (SPEC-literal), 1: pressure-mass preconditioned (default) */
  int smoother_fused; /* 1: fused halo-residual patch kernel (k <= 3), 0: one residual
                         launch per colour (default) */
} smg_config;

/* ---- context (replaces the reference's per-level setup: build_hierarchy mesh.hpp:30-36, the 1D
 *      matrix cache SPEC.md:157, fast_diag_prepare SPEC.md:338, coarse pseudo-inverse SPEC.md:468) */
int smg_config_default(smg_config* cfg);
int smg_create(const smg_config* cfg, smg_context** ctx);
int smg_destroy(smg_context* ctx);
int smg_set_stream(smg_context* ctx, void* cuda_stream); /* NULL = legacy default stream */
const char* smg_last_error(const smg_context* ctx);
/* number of CUDA kernels this context has launched so far (evidence counter for benchmarks) */
int64_t smg_launch_count(const smg_context* ctx);

/* ---- level layout (DoFLayout; BlockVector sizes block_vector.hpp:21-24) ---- */
/* sizes[0..2] velocity component blocks, sizes[3] pressure, sizes[4] total stored DoFs */
int smg_level_sizes(int degree, int level, int64_t sizes[5]);
/* w[a] = integral of the pressure nodal basis function a over the reference cell [0,1], a = 0..degree:
 * the separable weights of the mass-weighted pressure mean (project_zero_mean SPEC.md:212-220), for
 * callers that reduce the mean over a partitioned vector themselves */
int smg_pressure_node_weights(int degree, double* w);

/* ---- level vectors (device) ---- */
int smg_vec_alloc(smg_context* ctx, int level, int precision, void** dptr);
int smg_vec_free(smg_context* ctx, void* dptr);

/* ---- operator: y = A x, A = [[A, B^T],[B, 0]] (apply_stokes; Alg. 1)
 *      constrained (boundary-normal) rows of y are zero; constrained entries of x are ignored. */
int smg_vmult(smg_context* ctx, int level, int precision, void* y, const void* x);
/* r = b - A x (the residual of SPEC.md:424 / v_cycle SPEC.md:462) */
int smg_residual(smg_context* ctx, int level, int precision, void* r, const void* b, const void* x);

/* ---- smoother: one colour-by-colour multiplicative vertex-patch step on x (smooth SPEC.md:400-408,
 *      Alg. 2, local solver schur_solve SPEC.md:356-364). zero_init: x := 0 first. */
int smg_smooth(smg_context* ctx, int level, int precision, void* x, const void* b, int zero_init);

/* counters of the patch smoother since context creation or the last reset: patches solved and inner
 * Schur-CG iterations summed over them (mean iterations = cg_iterations / patches); synchronous */
int smg_smoother_stats(smg_context* ctx, int reset, int64_t* patches, int64_t* cg_iterations);

/* ---- transfer (prolongate / restrict SPEC.md:441-458): x_f += P x_c ;  r_c = P^T r_f ---- */
int smg_prolongate_add(smg_context* ctx, int coarse_level, int precision, void* x_fine, const void* x_coarse);
int smg_restrict(smg_context* ctx, int coarse_level, int precision, void* r_coarse, const void* r_fine);
/* level-0 pseudo-inverse apply (coarse_solve SPEC.md:468-476) */
int smg_coarse_solve(smg_context* ctx, int precision, void* x, const void* b);

/* ---- multigrid / Krylov callers (v_cycle SPEC.md:459-467; fgmres/solve_mixed SPEC.md:507-533) ---- */
int smg_vcycle(smg_context* ctx, int level, int precision, void* x, const void* b);
/* FGMRES(apply_A = fp64 vmult, apply_P = V-cycle in `vcycle_precision`) from x0 = 0; x, b fp64 device.
 * iters (out), history (out, max_iter+1 residual norms, may be NULL). Returns SMG_ENOTCONV if the
 * relative residual did not reach rel_tol. */
int smg_solve(smg_context* ctx, int level, void* x, const void* b, double rel_tol, int max_iter,
              int vcycle_precision, int* iters, double* history);

/* ---- z-slab partition (multi-GPU, one context per GPU). A slab vector holds the cells
 *      [max(z0-1,0), min(z1+1,m)) of the level: the owned cells [z0, z1) plus one ghost cell layer on
 *      each interior side; every block keeps its global x/y extents and the z node planes of those
 *      cells (u_z: the planes zlo(k+1) .. zhi(k+1) inclusive). The caller refreshes the ghost layers
 *      (halo exchange) before each apply; the operator writes the rows of the owned cells only.
 *      z1 - z0 must be a multiple of the kernel's brick depth (1, 2 or 4; use multiples of 4) unless
 *      z1 == m. ---- */
int smg_slab_sizes(int degree, int level, int z0, int z1, int64_t sizes[5]);
int smg_vmult_slab(smg_context* ctx, int level, int precision, void* y, const void* x, int z0, int z1);
int smg_residual_slab(smg_context* ctx, int level, int precision, void* r, const void* b, const void* x, int z0,
                      int z1);
/* ---- multigrid on z-slabs (general held ranges). A "held" vector holds the cells [zlo, zhi) of its
 *      level in the slab layout above; each call computes only the rows named by its cell range:
 *        residual_held       r = b - A x on the rows of cells [c0, c1) (held must cover c0-1 .. c1)
 *        smooth_colour_held  the patches of one colour whose vertex z plane is in [vz0, vz1]
 *        prolongate_add_held fine rows of fine cells [f0, f1) += P x_c
 *        restrict_held       coarse rows of coarse cells [c0, c1) = P^T r_f (reads fine cells 2c0-2 .. 2c1-1)
 *        dot_held            dot over the rows of cells [c0, c1) (fp64 accumulate; caller all-reduces) ---- */
int smg_held_sizes(int degree, int level, int zlo, int zhi, int64_t sizes[5]);
int smg_residual_held(smg_context* ctx, int level, int precision, void* r, const void* b, const void* x, int zlo,
                      int zhi, int c0, int c1);
int smg_smooth_colour_held(smg_context* ctx, int level, int precision, int colour, void* x, const void* r, int zlo,
                           int zhi, int vz0, int vz1);
int smg_prolongate_add_held(smg_context* ctx, int coarse_level, int precision, void* x_fine, const void* x_coarse,
                            int fzlo, int fzhi, int czlo, int czhi, int f0, int f1);
int smg_restrict_held(smg_context* ctx, int coarse_level, int precision, void* r_coarse, const void* r_fine, int fzlo,
                      int fzhi, int czlo, int czhi, int c0, int c1);
int smg_dot_held(smg_context* ctx, int level, int precision, const void* a, const void* b, int zlo, int zhi, int c0,
                 int c1, double* out);

/* dot over the owned rows of two slab vectors (fp64 accumulate); the caller all-reduces across ranks */
int smg_dot_slab(smg_context* ctx, int level, int precision, const void* a, const void* b, int z0, int z1,
                 double* out);

/* ---- multi-GPU driver (one context per GPU / rank; z-slab partition). The C form of the
 *      reference's seams for a partitioned mesh: fgmres(apply_A, apply_P, ...) and
 *      v_cycle. The ghost exchange and the reductions go through NCCL
 *      (smg_dist_init_nccl; rank 0 creates the id with smg_nccl_unique_id and the caller distributes it)
 *      or through caller callbacks (smg_dist_init_transport: MPI, torch.distributed, ...). All traffic is
 *      ordered on the context's stream. Distributed vectors use the HELD layout of smg_dist_held: the
 *      owned cells [z0, z1) of the rank plus 3 ghost cell layers per interior side (zlo, zhi); only the
 *      owned rows of inputs need to be valid. ---- */
typedef struct {
  /* post the given device->device messages between ranks (send[i] to rank send_peer[i], receive into
   * recv[i] from recv_peer[i]); stream-ordered on `stream` (cudaStream_t); 0 on success */
  int (*exchange)(void* user, int nsend, const void* const* send_ptr, const size_t* send_bytes,
                  const int* send_peer, int nrecv, void* const* recv_ptr, const size_t* recv_bytes,
                  const int* recv_peer, void* stream);
  /* in-place sum over the ranks of `count` device values (precision SMG_F64 / SMG_F32) */
  int (*allreduce_sum)(void* user, void* dev_values, size_t count, int precision, void* stream);
  void* user;
} smg_transport;
int smg_nccl_unique_id(char id[128]);
int smg_dist_init_nccl(smg_context* ctx, const char id[128], int nranks, int rank);
int smg_dist_init_transport(smg_context* ctx, const smg_transport* transport, int nranks, int rank);
/* owned cells [z0, z1) of `rank` on `level` (the partition every rank uses) */
int smg_dist_partition(int level, int nranks, int rank, int* z0, int* z1);
/* cells = {z0, z1, zlo, zhi} (owned, held) and sizes (held layout) of this rank's vectors on `level` */
int smg_dist_held(smg_context* ctx, int level, int cells[4], int64_t sizes[5]);
/* y = A x on the owned rows (x's ghost layers are exchanged first) */
int smg_dist_vmult(smg_context* ctx, int level, int precision, void* y, void* x);
/* dot over the owned rows, summed over the ranks (synchronous) */
int smg_dist_dot(smg_context* ctx, int level, int precision, const void* a, const void* b, double* out);
/* x = V-cycle(b) on the finest level (levels too thin to split are agglomerated and run replicated) */
int smg_dist_vcycle(smg_context* ctx, int precision, void* x, const void* b);
/* MG-preconditioned FGMRES over the slabs, smg_solve semantics (mass-weighted pressure mean removed) */
int smg_dist_solve(smg_context* ctx, void* x, const void* b, double rel_tol, int max_iter, int vcycle_precision,
                   int* iters, double* history);

/* ---- BLAS-1 on level vectors (block_vector.hpp:52-93); dots accumulate in fp64 ---- */
int smg_dot(smg_context* ctx, int level, int precision, const void* a, const void* b, double* out);
int smg_axpy(smg_context* ctx, int level, int precision, double alpha, const void* x, void* y);
int smg_convert(smg_context* ctx, int level, int dst_precision, void* dst, int src_precision, const void* src);
/* x *= alpha (scale, block_vector.hpp:74-78) */
int smg_scale(smg_context* ctx, int level, int precision, double alpha, void* x);
/* y = b - y (subtract_from, block_vector.hpp:80-88: residuals computed in place) */
int smg_subtract_from(smg_context* ctx, int level, int precision, const void* b, void* y);
/* sqrt(dot(x, x)) with fp64 accumulation (norm, block_vector.hpp:63-66); synchronous */
int smg_norm(smg_context* ctx, int level, int precision, const void* x, double* out);
/* subtract the mass-weighted mean of the pressure block so that int p_h dx = 0
 * (project_zero_mean); velocity blocks untouched */
int smg_project_zero_mean(smg_context* ctx, int level, int precision, void* x);

/* ---- host BlockVector <-> device level vector (BlockVector<dim,T> block_vector.hpp:15-18 with the
 *      DoFLayout of SPEC.md:173-176: velocity component blocks lexicographic x-fastest including the
 *      constrained boundary-normal DoFs; pressure CELL-LOCAL lexicographic, i.e. cells x-fastest and
 *      (k+1)^3 nodes per cell x-fastest). Host arrays are caller-owned; synchronous. ---- */
int smg_vec_upload(smg_context* ctx, int level, int precision, void* dst, const void* const vel[3], const void* p);
int smg_vec_download(smg_context* ctx, int level, int precision, void* const vel[3], void* p, const void* src);

/* ---- host-buffer operator apply in the BlockVector layout (the reference-facing vmult: what
 *      StokesOperator::vmult(BlockVector&, const BlockVector&) becomes; copies included) ---- */
int smg_vmult_host(smg_context* ctx, int level, int precision, void* const y_vel[3], void* y_p,
                   const void* const x_vel[3], const void* x_p);

#ifdef __cplusplus
}
#endif

#endif /* SMG_B200_H */
