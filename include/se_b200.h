/*
 * se_b200.h -- C ABI of the B200-native Spectral Ewald (SE) hot path.
 *
 * Drop-in boundary for the reference package `pmewald` (arXiv 1712.04732,
 * /root/reference/pkg/src/pmewald).  Every entry point names the reference
 * interface it replaces (file:line).  Plain pointers and sizes only; no
 * torch / numpy types.  All compute runs in hand-written sm_100a CUDA
 * kernels plus cuFFT; there is no CPU fallback for any compute entry point.
 *
 * Conventions
 *  - Positions are (N,3) row-major float64 ("AoS", as ParticleSystem.positions,
 *    core.py:57-86); charges and potentials are (N,) float64.
 *  - Grids use the reference's numpy layout: C order [ix][iy][iz] of
 *    Grid.shape (sekspace.py:64-66): M on periodic axes, Mt = M + P on free
 *    axes; the first D axes are periodic (core.py:44-46).
 *  - Functions suffixed _dev take DEVICE pointers (on the plan's device and
 *    ordered on the plan's stream); functions suffixed _host take HOST
 *    pointers and include the host<->device copies.
 *  - Every call returns an int status; SE_OK == 0.  se_last_error() returns
 *    the thread-local message of the last failure.  Status -> Python
 *    exception mapping (core.py:23-28):
 *        SE_EINVAL    -> ValueError
 *        SE_ECONFIG   -> ConfigurationError(ValueError)
 *        SE_ESINGULAR -> SingularConfigurationError(ValueError)
 *        SE_ENUMERIC  -> AssertionError   (numerical guards)
 *        SE_EDEVICE   -> RuntimeError     (CUDA / cuFFT failure, no device)
 */
#ifndef SE_B200_H
#define SE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SE_OK 0
#define SE_EINVAL 1
#define SE_ECONFIG 2
#define SE_ESINGULAR 3
#define SE_ENUMERIC 4
#define SE_EDEVICE 5

/* window kinds: windows.py:24-27 ("gaussian", "kb", "bm") */
#define SE_WINDOW_GAUSSIAN 0
#define SE_WINDOW_KB 1
#define SE_WINDOW_BM 2

/* timings[] slots, the reference's stage keys (sekspace.py:359-388, core.py:211-213) */
#define SE_T_REALSPACE 0
#define SE_T_SPREAD 1
#define SE_T_AFT 2
#define SE_T_SCALE 3
#define SE_T_AIFT 4
#define SE_T_GATHER 5
#define SE_T_PRECOMPUTE 6
#define SE_T_COUNT 7

/* SEParams (core.py:89-116), field for field. */
typedef struct se_params {
    double xi;      /* Ewald splitting parameter */
    double rc;      /* real-space cutoff */
    int32_t M;      /* grid points per periodic axis (even) */
    int32_t P;      /* window support points */
    int32_t window; /* SE_WINDOW_* */
    int32_t nI;     /* low-mode block half width (D in {1,2}) */
    double shape;   /* m (gaussian) or beta (kb, bm) */
    double s0;      /* zero-block upsampling */
    double s;       /* I-block upsampling */
    double R;       /* truncation radius of the free-space kernel (D < 3) */
    double eps;     /* accuracy target the set was built for */
} se_params_t;

/* Grid (sekspace.py:36-70) as built by Grid.build for (L, params, D). */
typedef struct se_grid {
    int32_t D, M, P, Mt, g0, gs;
    int32_t shape[3];
    double L, h, Lt, R;
    double offsets[3];
} se_grid_t;

typedef struct se_plan *se_plan_t;

/* ------------------------------------------------------------------ *
 * Host-side planning (no device needed).                              *
 * ------------------------------------------------------------------ */

/* SEParams.validate (core.py:118-138).  SE_EINVAL with the reference's message. */
int se_params_validate(const se_params_t *p, double L, int D);
/* Grid.build (sekspace.py:53-62). */
int se_grid_build(int D, double L, const se_params_t *p, se_grid_t *out);
/* aft.padded_size (aft.py:76-84) and aft.next_even_smooth (aft.py:68-73). */
int se_padded_size(double s, int32_t n, int32_t *out);
int se_next_even_smooth(int32_t n, int32_t *out);
/* The real-space kernel's polynomial pair term for (xi, rc): erfc(xi r)/r =
 * 1/r - Q(r^2) (kind 0, potential) or (erfc(xi r)/r + 2 xi/sqrt(pi)
 * exp(-xi^2 r^2))/r^2 = (1/r - R(r^2))/r^2 (kind 1, field), Q / R =
 * sum_i coeffs[i] t^i, t = 2 r^2 / rc^2 - 1 (replaces the erfc of
 * realspace.py:123-126 inside the kernel).  coeffs: 33 doubles; *degree =
 * 20..32, or 0 when no degree <= 32 reaches the kernel's accuracy (xi rc >
 * ~5: the kernel then evaluates erfc directly). */
int se_pair_poly_coefficients(double xi, double rc, int kind, double *coeffs, int32_t *degree);
/* precompute_truncated_greens geometry (sekspace.py:266-279): nconv, fine g0, R. */
int se_d0_kernel_geometry(double L, int32_t M, int32_t P, double s0, double rc,
                          int32_t *nconv, int32_t *g0, double *R);
/* Mode partition counts of ModePartition.build (aft.py:102-117). */
int se_mode_partition_counts(int32_t M, int D, int32_t nI, int64_t *nI_rows, int64_t *nJ_rows);
/* Window tables used by the plan (windows.py:242-257): real-space values and
 * Fourier transforms (BM by long-double Gauss-Legendre quadrature,
 * windows.py:175-239).  h is the grid spacing, w = P*h/2. */
int se_window_eval(int window, int32_t P, double h, double shape,
                   const double *x, int64_t n, double *out);
int se_window_fourier(int window, int32_t P, double h, double shape,
                      const double *k, int64_t n, double *out);
/* The two numerical kernels behind the transforms above: the BM transform
 * by an n-node long-double Gauss-Legendre rule in theta (windows.py:202-211,
 * `_bm_quadrature`) and the KB transform's sinh(r)/r continued to rho2 < 0
 * (windows.py:115-132, `_sinhc`). */
int se_bm_quadrature(double w, double beta, const double *k, int64_t n, int32_t nodes, double *out);
int se_kb_sinhc(const double *rho2, int64_t n, double *out);
/* realspace.build_cell_list (realspace.py:43-59): n^3 cells of edge L/n;
 * order[bounds[c] .. bounds[c+1]) are the particles of flat cell
 * c = (cx*n + cy)*n + cz in ascending index order.  order: N, bounds: n^3+1.
 * Inspection utility; the device kernels bin on their own finer grid. */
int se_cell_list_host(const double *pos, int64_t N, double L, int32_t n, int64_t *order, int64_t *bounds);
/* greens.zero_mode_values (greens.py:48-85). */
int se_greens_zero_mode(int D, double R, const double *kappa, int64_t n, double *out);

/* ------------------------------------------------------------------ *
 * Plan: device resources (tables, cuFFT plans, D=0 kernel, buffers).   *
 * Mirrors the reference's caches (sekspace.py:97, windows.py:169-172). *
 * ------------------------------------------------------------------ */

/* Validate (core.py:118-138), build the grid (sekspace.py:53-62) and bind
 * the plan to `device`.  Tables / FFT plans are created on first use. */
int se_plan_create(se_plan_t *plan, int D, double L, const se_params_t *p, int device);
int se_plan_destroy(se_plan_t plan);
/* Stream for all subsequent calls (cudaStream_t; 0 = the legacy default
 * stream).  Until it is called the plan uses a stream of its own. */
int se_plan_set_stream(se_plan_t plan, void *stream);
int se_plan_grid(se_plan_t plan, se_grid_t *out);
/* CUDA graphs for the fused total potential (default on): repeated calls
 * with the same (pos, q, phi, N, stream) replay one graph of the device work
 * (first call eager, second call captured).  0 = always launch eagerly. */
int se_plan_set_graphs(se_plan_t plan, int on);
/* Deferred checks (on != 0): the shard entry points (se_*_shard_dev,
 * se_kspace_apply_dev) only enqueue work -- no host synchronisation for the
 * device error flags or profiling events -- so one host thread can keep
 * several streams busy; se_plan_finish synchronises the plan's stream, raises
 * a pending error (coincident particles -> SE_ESINGULAR) and collects the
 * profiling events. */
int se_plan_set_deferred_checks(se_plan_t plan, int on);
/* Deterministic mode (on != 0; default from the environment variable
 * SE_B200_DETERMINISTIC at plan creation): results are bitwise reproducible
 * run to run, as the reference's thread-count independence requires
 * (test_core.py:139-145, test_realspace.py:129-133).  The real-space sum
 * then runs without Newton's third law (each target sums all its partners
 * itself, no source-side atomics; ~2x the pair work) and spreading writes
 * per-work-unit tiles that are reduced into the grid in a fixed order
 * (instead of fp64 atomic tile flushes).  The default mode agrees with it
 * to rounding (~1e-15 relative). */
int se_plan_set_deterministic(se_plan_t plan, int on);
int se_plan_finish(se_plan_t plan);
/* Number of kernel launches issued by this plan since creation (for the bench). */
int se_plan_launch_count(se_plan_t plan, int64_t *count);
/* Warning bits raised by the last total-potential call: bit 0 = the system is
 * not charge neutral in free space (core.py:185-189 warns instead of raising). */
int se_plan_warnings(se_plan_t plan, int *flags);
/* Per-kernel device timing of the hot kernels, for roofline reporting:
 * CUDA events recorded on the plan's stream around each launch when
 * profiling is on; times accumulate (ms) with launch counts per slot. */
#define SE_K_REALSPACE 0 /* real-space erfc pair kernel */
#define SE_K_SPREAD 1    /* spreading kernel */
#define SE_K_GATHER 2    /* gathering kernel */
#define SE_K_KSPACE 3    /* k-space stage (cuFFT + multiplier kernels) */
#define SE_K_SORT 4      /* particle binning (keys, radix sort, records, units) */
#define SE_K_COUNT 5
int se_plan_set_profiling(se_plan_t plan, int on);
int se_plan_kernel_times(se_plan_t plan, double *ms, int64_t *launches);
/* Number of ordered in-cutoff pairs (r < rc, r >= 1e-14) the real-space sum
 * evaluates: the unit of the real-space roofline (cell path only). */
int se_realspace_pair_count_dev(se_plan_t plan, const double *pos, const double *q, int64_t N,
                                int64_t *pairs);
/* Truncated-kernel geometry the plan uses for D = 0 (sekspace.py:266-279). */
int se_plan_d0_geometry(se_plan_t plan, int32_t *nconv, int32_t *g0, double *R);

/* ParticleSystem / check_neutrality validation on device arrays (core.py:65-77,
 * 180-191): SE_EINVAL if a coordinate lies outside [0, L); with neutrality
 * != 0 (and q non-null) also SE_EINVAL for a non-neutral periodic system
 * (D = 0: warning bit 0, see se_plan_warnings).  The _dev stage entry points
 * run the box check themselves; the shard entry points do so unless
 * deferred checks are on, in which case the caller checks once per call
 * (paper_1712_04732_b200.distributed does). */
int se_check_system_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, int neutrality);

/* sekspace.spread (sekspace.py:130-156): grid = sum_n q_n w (x) w (x) w.
 * grid_out holds prod(Grid.shape) float64 and is overwritten. */
int se_spread_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *grid_out);
/* aft_forward -> scale -> aft_inverse -> real part (sekspace.py:369-381), or the
 * D=0 precomputed-kernel path _kspace_freespace_kernel (sekspace.py:301-337)
 * when D == 0 and use_kernel != 0.  In place on a Grid.shape float64 grid. */
int se_kspace_apply_dev(se_plan_t plan, double *grid, int use_kernel, double *timings);
/* sekspace.gather (sekspace.py:159-178), including the h^3 weight.
 * accumulate != 0 adds into phi instead of overwriting. */
int se_gather_dev(se_plan_t plan, const double *grid, const double *pos, int64_t N,
                  double *phi, int accumulate);
/* sekspace.se_kspace (sekspace.py:340-389): spread, k-space stage, gather. */
int se_kspace_potential_dev(se_plan_t plan, const double *pos, const double *q, int64_t N,
                            double *phi, int use_kernel, double *timings);
/* realspace.real_space_sum (realspace.py:168-180); add_self != 0 also adds
 * realspace.self_term (realspace.py:183-185).  SE_ESINGULAR on coincident
 * particles (realspace.py:121-122,157,161). */
int se_realspace_dev(se_plan_t plan, const double *pos, const double *q, int64_t N,
                     double *phi, int add_self);
/* core.total_potential (core.py:194-216): phi = phi_R + phi_F + phi_self.
 * Input errors (coordinates outside [0, L), core.py:65-77; a non-neutral
 * periodic system, core.py:180-191; coincident particles) are returned as
 * SE_EINVAL / SE_ESINGULAR like everywhere else, but are detected by a check
 * kernel INSIDE the device work and read back with one synchronisation at
 * the end of the call -- phi is undefined when the status is not SE_OK. */
int se_total_potential_dev(se_plan_t plan, const double *pos, const double *q, int64_t N,
                           double *phi, double *timings);

/* Sharded variants for one-process-per-GPU runs: every rank holds all N
 * particles; rank r of `world` computes the share of particles it owns
 * (a contiguous range of the cell-sorted order) and writes only those
 * entries of phi (others are zeroed), so a sum-all-reduce of phi over
 * ranks gives core.total_potential.  The spread grid of a shard is partial:
 * the caller sum-all-reduces it before se_kspace_apply_dev. */
int se_spread_shard_dev(se_plan_t plan, const double *pos, const double *q, int64_t N,
                        int rank, int world, double *grid_out);
int se_gather_shard_dev(se_plan_t plan, const double *grid, const double *pos, int64_t N,
                        int rank, int world, double *phi, int accumulate);
int se_realspace_shard_dev(se_plan_t plan, const double *pos, const double *q, int64_t N,
                           int rank, int world, double *phi, int add_self);

/* Domain-decomposed real space (particles partitioned over ranks by x-slabs
 * of columns; paper_1712_04732_b200.distributed.total_potential_domain).
 * The column grid is ncols x ncols columns in (x, y) of edge L / ncols >=
 * rc / 3, identical on every rank; this rank owns the columns with
 * cx in [col_lo, col_hi).  The local set is pos/q[0, n_own) = the own
 * particles (exactly those in the own columns, column index floor(x / edge)
 * clamped to [0, ncols - 1]) followed by pos/q[n_own, n_local) = the halo:
 * every particle of the ceil(rc ncols / L) columns beyond col_hi (+x side,
 * wrapping on a periodic x).  Each unordered in-cutoff pair with an own end
 * is evaluated once over all ranks (half shell towards +x, Newton's third
 * law).  phi[0, n_own) = the real-space potentials of the own particles
 * (+ self term if add_self), phi[n_own, n_local) = the source-side partial
 * sums of the halo particles, which the caller returns to their owners.
 * Needs rc <= L / 2 and >= 2 reach + 1 columns per periodic axis. */
int se_realspace_domain_dev(se_plan_t plan, const double *pos, const double *q, int64_t n_local, int64_t n_own,
                            int ncols, int col_lo, int col_hi, double *phi, int add_self);

/* Electric field E = -grad phi at every particle (forces F = q E; the
 * reference stops at potentials: SPEC.md:16 notes the force integration "has
 * to be performed three times").  E is (N, 3) in caller
 * order: the real-space pair field q_s (erfc(xi r)/r + 2 xi/sqrt(pi)
 * exp(-xi^2 r^2)) (x_t - x_s)/r^2 over the same pair set as
 * real_space_sum, plus the Fourier field: D = 3 gathered from the
 * spectrally differentiated grid (-i k times the scaled spectrum, one
 * inverse transform and one gather per component); D < 3 the gradient of
 * the gather on the filtered grid of the potential (window derivative;
 * SE_EINVAL for the ES window, whose derivative is singular at the support
 * edge).  No self term (the self-interaction is a constant).  Errors as
 * se_total_potential_*. */
int se_total_field_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E);
int se_total_field_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E);
/* The two parts separately (host pointers): the real-space pair field (any
 * D; the same pair set as real_space_sum) and the Fourier field. */
int se_realspace_field_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E);
int se_kspace_field_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E);

/* Slab-decomposed k-space stage of D = 3 (aft.py:203-206 + sekspace.py:198-206
 * + aft.py:237-238 split over `world` ranks).  Rank r owns the
 * x-slab of nx = M / world planes (block r of the C-order grid, as a
 * reduce-scatter leaves it); M % world == 0.  Also D = 0 on the truncated-
 * kernel path (_kspace_freespace_kernel, sekspace.py:301-337): the transform
 * size is then nconv (se_plan_d0_geometry), nx = nconv / world padded
 * x-planes per rank, and the slab buffers hold the (nx, Mt, Mt) planes of
 * the Mt^3 spread grid (planes >= Mt are zero), zero-padded / restricted
 * inside.  Complex buffers are interleaved fp64 (re, im):
 *   se_slab_forward_dev: slab (nx, M, M) real -> send (world, nx, nky, nkz)
 *     complex: 2-D R2C over (y, z), block s = this rank's planes x ky-chunk s;
 *   (caller: all-to-all of equal blocks -> recv, i.e. (M, nky, nkz) = all kx
 *     of this rank's ky-chunk)
 *   se_slab_xpass_dev: in place on recv: x-FFT, Green's-function / window
 *     multiplier (x 1/M^3), inverse x-FFT;
 *   (caller: all-to-all back)
 *   se_slab_inverse_dev: back (world, nx, nky, nkz) -> slab (nx, M, M) real
 *     (the slab of the k-space-filtered grid; an all-gather gives the grid).
 * se_slab_geometry returns nx, nky = n / world and nkz = n / 2 + 1 (n = M, or
 * nconv for D = 0). */
int se_slab_geometry(se_plan_t plan, int world, int64_t *nx, int64_t *nky, int64_t *nkz);

/* Row-distributed adaptive FFT of D = 1, 2 (aft.py:168-265 + sekspace.py:217-254
 * split over `world` ranks).  Rank r holds the z-chunk
 * z in [nz0, nz0 + nz), nz0 = Mt r / world, of the grid (every x, y): the
 * periodic R2C is local to z-planes, its rows (periodic modes: (kx, ky < M/2+1)
 * for D = 2 in chunks of M / world kx values, kx < M/2+1 for D = 1 in chunks of
 * ceil((M/2+1) / world)) are grouped by chunk, and an all-to-all gives each rank
 * every z of its rows, where the zero / I / J free-axis blocks are padded,
 * transformed, scaled and inverted as in se_kspace_apply_dev.  Complex buffers
 * are interleaved fp64:
 *   se_zslab_geometry: out6 = {nz0, nz, row0, nrows, rows_total, per_y} (a row
 *     carries per_y x (z) values: per_y = 1 for D = 2, Mt for D = 1);
 *   se_zslab_forward_dev: zslab (M, M or Mt, nz) real -> spec (rows_total,
 *     per_y, nz): rows of rank d's chunk are contiguous (the all-to-all's send
 *     blocks: nrows_d x per_y x nz values to rank d);
 *   se_zslab_rows_dev: in place on recv = (source s) x (nrows, per_y, nz_s):
 *     this rank's rows through the free-axis blocks;
 *   se_zslab_inverse_dev: spec (rows_total, per_y, nz) -> zslab real (the
 *     spectrum is used as scratch). */
int se_zslab_geometry(se_plan_t plan, int world, int rank, int64_t *out6);
int se_zslab_forward_dev(se_plan_t plan, int world, int rank, const double *zslab, double *spec);
int se_zslab_rows_dev(se_plan_t plan, int world, int rank, double *recv);
int se_zslab_inverse_dev(se_plan_t plan, int world, int rank, const double *spec, double *zslab);
int se_slab_forward_dev(se_plan_t plan, int world, const double *slab, double *send);
int se_slab_xpass_dev(se_plan_t plan, int world, int rank, double *recv);
int se_slab_inverse_dev(se_plan_t plan, int world, const double *back, double *slab);

/* realspace.self_term (realspace.py:183-185): out = -2 xi q / sqrt(pi), on the
 * current CUDA device.  _dev: device pointers on `stream` (cudaStream_t). */
int se_self_term_dev(const double *q, int64_t N, double xi, double *out, void *stream);
int se_self_term_host(const double *q, int64_t N, double xi, double *out);

/* core.total_potential through HOST buffers: H2D copies of pos/q, the device
 * pipeline, and the D2H copy of phi, all on the plan's stream. */
int se_total_potential_host(se_plan_t plan, const double *pos, const double *q, int64_t N,
                            double *phi, double *timings);
/* sekspace.se_kspace / spread / gather / real_space_sum through host buffers. */
int se_kspace_potential_host(se_plan_t plan, const double *pos, const double *q, int64_t N,
                             double *phi, int use_kernel, double *timings);
int se_spread_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *grid_out);
int se_gather_host(se_plan_t plan, const double *grid, const double *pos, int64_t N, double *phi);
int se_kspace_apply_host(se_plan_t plan, double *grid, int use_kernel);
int se_realspace_host(se_plan_t plan, const double *pos, const double *q, int64_t N,
                      double *phi, int add_self);

/* precompute_truncated_greens (sekspace.py:257-298): the real half-spectrum
 * table (nconv, nconv, nconv/2+1), computed on the device and copied to host
 * (`out` must hold nconv*nconv*(nconv/2+1) doubles). */
int se_d0_kernel_table_host(se_plan_t plan, double *out);

/* ------------------------------------------------------------------ *
 * Stage-level API of the reference (aft.py / sekspace.scale).         *
 * ------------------------------------------------------------------ */

/* The FFT-engine plugin (aft.py:24-53, numpy semantics) on cuFFT, for a
 * C-ordered array of `ndim` dims and the contiguous axis block [ax0, ax1];
 * complex data are interleaved (re, im) doubles.  c2c: same shape in and
 * out, inverse carries 1/n.  r2c: real `shape` in, the last transformed axis
 * becomes n/2+1.  c2r: `out_shape` is the real output shape, 1/n included.
 * Host pointers; `device` selects the GPU. */
int se_fft_c2c_host(int device, int ndim, const int64_t *shape, int ax0, int ax1, int inverse,
                    const double *in, double *out);
int se_fft_r2c_host(int device, int ndim, const int64_t *shape, int ax0, int ax1,
                    const double *in, double *out);
int se_fft_c2r_host(int device, int ndim, const int64_t *out_shape, int ax0, int ax1,
                    const double *in, double *out);
/* sekspace.scale (sekspace.py:192-254) in place on a SpectralField's blocks
 * (aft.py:124-152): D=3 `full` (M^3) or D=0 `zero` (g0^3) in cube_or_zero;
 * D in {1,2}: zero block, I rows (gs^{3-D} each) with I_idx (nI x D periodic
 * mode indices) and J rows (Mt^{3-D}) with J_idx.  kp/wp, k0/w0, ks/ws,
 * kt/wt: wavenumbers and window transforms on the M, g0, gs and Mt mode sets. */
int se_scale_blocks_host(int device, int D, int M, int Mt, int g0, int gs, double xi, double R,
                         const double *kp, const double *wp, const double *k0, const double *w0,
                         const double *ks, const double *ws, const double *kt, const double *wt,
                         double *cube_or_zero, double *Iblk, const int *I_idx, int64_t nI,
                         double *Jblk, const int *J_idx, int64_t nJ);

/* ------------------------------------------------------------------ *
 * Direct Ewald sums (the reference's oracle.py evaluators) on the      *
 * device, for validating the SE path at full size.  pos (N,3) AoS, q   *
 * (N,); targets = indices into the system (NULL: all N, T ignored);    *
 * phi has T (resp. N) entries.  _dev: device pointers, synchronous on  *
 * `stream`; _host: host buffers.                                       *
 * ------------------------------------------------------------------ */
/* oracle.kspace_direct_3p (oracle.py:109-118): Fourier-space Ewald sum over
 * the integer modes |n_a| <= kmax, n != 0. */
int se_direct_kspace_3p_dev(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                            const int64_t *targets, int64_t T, double *phi, void *stream);
int se_direct_kspace_3p_host(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                             const int64_t *targets, int64_t T, double *phi);
/* oracle.kspace_direct_2p (oracle.py:120-153): closed-form doubly periodic
 * Fourier sum over the modes |n_a| <= kmax of the periodic axes (x, y). */
int se_direct_kspace_2p_dev(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                            const int64_t *targets, int64_t T, double *phi, void *stream);
int se_direct_kspace_2p_host(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                             const int64_t *targets, int64_t T, double *phi);
/* oracle.kspace_direct_1p (oracle.py:156-178): singly periodic Fourier sum
 * (incomplete Bessel K0 per mode, log + E1 zero mode); periodic axis x.
 * SE_ESINGULAR if two charges share transverse coordinates. */
int se_direct_kspace_1p_dev(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                            const int64_t *targets, int64_t T, double *phi, void *stream);
int se_direct_kspace_1p_host(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                             const int64_t *targets, int64_t T, double *phi);
/* oracle.kspace_direct_0p (oracle.py:181-192): sum_{n != m} q_n erf(xi r)/r
 * + q_m 2 xi / sqrt(pi); SE_ESINGULAR for coincident distinct particles. */
int se_direct_kspace_0p_dev(const double *pos, const double *q, int64_t N, double xi, const int64_t *targets,
                            int64_t T, double *phi, void *stream);
int se_direct_kspace_0p_host(const double *pos, const double *q, int64_t N, double xi, const int64_t *targets,
                             int64_t T, double *phi);

/* Thread-local message of the last failing call. */
const char *se_last_error(void);
/* Library version string. */
const char *se_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SE_B200_H */
