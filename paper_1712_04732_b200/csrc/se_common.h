// Internal declarations shared by the SE B200 library translation units.
#pragma once
#include <atomic>

#include <cuda_runtime.h>
#include <cufft.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/se_b200.h"

namespace se {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error(code, msg); }

void set_last_error(const std::string &msg);

#define SE_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            ::se::fail(SE_EDEVICE, std::string("CUDA error: ") + cudaGetErrorString(e_) \
                                       + " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define SE_CUFFT(call)                                                                  \
    do {                                                                                \
        cufftResult r_ = (call);                                                        \
        if (r_ != CUFFT_SUCCESS)                                                        \
            ::se::fail(SE_EDEVICE, std::string("cuFFT error ") + std::to_string((int)r_) \
                                       + " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define SE_LAUNCH_CHECK() SE_CUDA(cudaGetLastError())

// ------------------------------------------------------------ host planning
int padded_size(double s, int n);
int next_even_smooth(int n);
void validate(const se_params_t &p, double L, int D);
se_grid_t build_grid(int D, double L, const se_params_t &p);
struct D0Geom { int nconv, g0; double R; };
D0Geom d0_geometry(double L, int M, int P, double s0, double rc, bool has_rc);
std::vector<int> signed_modes(int n);
std::vector<double> wavenumbers(int n, double h);
// window Fourier transform at wavenumbers k (windows.py:251-257); BM uses the
// long-double quadrature of windows.py:175-239.
std::vector<double> window_fourier(int window, int P, double h, double shape,
                                   const std::vector<double> &k);
double window_value(int window, double w, double shape, double x);
double greens_zero_mode(int D, double R, double kappa);
// polynomial pair term of the real-space kernel: coefficients, degree (0: none) -- se_host.cpp
int pair_poly_fit(double xi, double rc, int kind, double *pc);
double bessel_i0(double x);

// ---------------------------------------------------------- device buffers
// Bumped on every device (re)allocation of a DevBuf: a captured CUDA graph
// is replayed only while no buffer it may reference has moved.
inline std::atomic<unsigned long long> g_buf_generation{0};

struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    void ensure(size_t n) {
        if (n <= bytes) return;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        g_buf_generation.fetch_add(1);
        if (n == 0) return;
        SE_CUDA(cudaMalloc(&ptr, n));
        bytes = n;
    }
    void release() {
        if (ptr) {
            cudaFree(ptr);
            g_buf_generation.fetch_add(1);
        }
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(ptr); }
};

// Per-axis mode table on the device: wavenumbers and window transforms.
struct ModeTable {
    int n = 0;
    DevBuf k, what;
};

// Particle binning: sort by a key and build (bin, start, count) work units.
struct Binning {
    int nbins = 0;
    int64_t capacity = 0;
    DevBuf keys, keys_sorted, idx, idx_sorted, counts, starts, units, nunits, ubstart;
    DevBuf fhist, fstart, bsum;  // counting sort: fine-bin histogram / starts, scan block sums
    DevBuf large, nlarge;        // counting sort: fine bins too large for the per-thread insertion sort
    DevBuf rec;  // sorted particle records (x, y, z, q) as double4
    int fine_shift = 0;          // index bits refining a coarse key
    int64_t nfine = 0;           // fine bins
};

struct TileGeom {
    int T;        // tile edge along x and y in start-index units
    int Tz;       // tile edge along z
    int Tp;       // padded x / y edge T + P - 1
    int pitch;    // padded z edge Tz + P - 1 (the z pitch of the smem tile, doubles)
    int nt[3];    // tiles per axis
    int lo[3];    // first start index per axis
    int nwarps;   // warps per CTA (x-plane owners)
    int batch;    // particles staged per batch
    size_t smem;  // dynamic shared memory bytes
};

struct CellGeom {
    int n;        // cells per axis
    double edge;  // cell edge
    int mode[3];  // 0: free (clip), 1: periodic wrap +-2, 2: periodic, all cells + min image
};

// Domain-decomposed real space (se_realspace_domain_dev): the column grid
// is fixed by the caller (the same on every rank), targets are the
// particles of the columns with cx in [col_lo, col_hi), the rest of the
// local set is +x halo (sources only); ncols = 0: the usual single-set sum.
struct DomainSpec {
    int ncols = 0, col_lo = 0, col_hi = 0;
    int64_t n_own = -1;  // caller-order particles [0, n_own) are the own ones
};

struct se_plan_impl;

}  // namespace se

struct se_plan {
    int D = 3;
    double L = 1.0;
    se_params_t p{};
    se_grid_t g{};
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    int64_t launches = 0;

    // spreading / gathering
    se::TileGeom tile{};
    se::Binning tbin;  // tile binning for spread / gather
    // real space
    se::CellGeom cell{};
    se::DomainSpec dom{};
    se::Binning cbin;  // cell binning for the real-space sum
    se::DevBuf flag;   // device error flags (int)
    se::DevBuf sdet;   // deterministic spreading: per-unit padded tiles

    // k-space
    bool kspace_ready = false;
    double xi_tables = -1.0;
    se::ModeTable tM, tg0, tgs, tMt, tNc, tNh;
    se::DevBuf spec, spec2, spec3, work, grid_tmp, rows_I;  // spectra / padded buffers
    int nI_rows = 0;  // half-plane I rows (D=2: pairs, D=1: planes)
    cufftHandle fft_fwd = 0, fft_inv = 0;           // main transforms
    cufftHandle fft_rowJ = 0, fft_rowI = 0, fft_row0 = 0;  // free-axis transforms (D in {1,2})
    bool fft_made = false;
    // D=0 kernel path
    bool d0_ready = false;
    int nconv = 0, kg0 = 0;
    double kR = 0.0;
    se::DevBuf ghat;
    cufftHandle fft_c_fwd = 0, fft_c_inv = 0;
    bool d0_fft_made = false;
    // D=0 full-upsampling path
    cufftHandle fft_f_fwd = 0, fft_f_inv = 0;
    bool d0full_fft_made = false;
    se::DevBuf grid_dev;  // scratch grid for the fused pipelines
    se::DevBuf io_pos, io_q, io_phi, io_grid;  // staging for _host calls
    se::DevBuf check;  // neutrality / box reduction scratch
    int warnings = 0;  // bit 0: non-neutral system in free space (core.py:185-189)
    // per-kernel CUDA-event timing of the hot kernels (bench roofline)
    bool prof = false;
    cudaEvent_t pev[SE_K_COUNT][2] = {};
    bool pending[SE_K_COUNT] = {};
    double pms[SE_K_COUNT] = {};
    int64_t pcount[SE_K_COUNT] = {};
    se::DevBuf pairs;  // pair counter (count mode of the real-space kernel)
    se::DevBuf racc;   // real-space pair sums in cell-sorted order (Newton path)
    // CUDA graph of the fused total-potential body (real space + spread +
    // k-space + gather), replayed for repeated calls with the same buffers
    bool graphs = true;
    // bitwise reproducible results (no order-dependent fp64 atomics): the
    // real-space sum without Newton's third law, spreading through per-unit
    // tiles reduced in a fixed order; from SE_B200_DETERMINISTIC at creation
    bool deterministic = false;
    // the real-space kernel's polynomial pair term (pair_poly_fit, ~1 ms of
    // host work): fitted once per (xi, rc, kind) and kept with the plan
    struct PairPoly {
        bool valid = false;
        double xi = 0.0, rc = 0.0;
        int deg = 0;
        double pc[33] = {};
    } pair_poly[2];  // kind 0: potential, 1: field
    cudaGraphExec_t gexec = nullptr;
    const void *gkey[3] = {};  // pos, q, phi
    int64_t gN = -1;
    cudaStream_t gstream = nullptr;
    bool gprof = false, gwarm = false;
    int64_t glaunches = 0;           // kernels per replay (for the launch counter)
    unsigned long long ggen = 0;     // DevBuf generation the graph was captured at
    bool gpending[SE_K_COUNT] = {};  // profiling slots recorded by the graph
    cudaEvent_t gfence[2] = {};      // orders the graph stream after / before a legacy caller stream
    bool capturing = false;          // inside graph capture: profiling events become record nodes
    // overlap of the k-space pipeline (side stream, higher priority) with the
    // real-space kernel in total_potential
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    se::DevBuf phik;  // phi_F of the overlapped k-space pipeline
    se::DevBuf fgrid, fphi, io_E;  // field: three filtered grids, three gathered components, host staging
    // slab-decomposed D = 3 k-space stage (per world size)
    int slab_world = 0;
    // deferred checks: the shard entry points return without synchronising
    // (device error flags, profiling events); se_plan_finish does both
    bool defer = false;
    double *verdict_host = nullptr;  // pinned: check sums [0..3], singularity flag [4] (total_verdict)
    cufftHandle slab_f2 = 0, slab_i2 = 0, slab_x = 0;
    // row-distributed AFT (D = 1, 2), for one (world, rank)
    int zs_world = -1, zs_rank = -1, zs_nI = 0;
    cufftHandle zs_fwd = 0, zs_inv = 0, zs_rowJ = 0, zs_rowI = 0, zs_row0 = 0;
    se::DevBuf zs_rowsI, zs_Hk, zs_Z, zs_B;
};

namespace se {

// per-kernel timing (no-ops unless the plan's profiling flag is set)
inline void prof_begin(se_plan *pl, int id) {
    if (!pl->prof) return;
    if (!pl->pev[id][0]) {
        SE_CUDA(cudaEventCreate(&pl->pev[id][0]));
        SE_CUDA(cudaEventCreate(&pl->pev[id][1]));
    }
    SE_CUDA(cudaEventRecordWithFlags(pl->pev[id][0], pl->stream,
                                     pl->capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
}
inline void prof_end(se_plan *pl, int id) {
    if (!pl->prof) return;
    SE_CUDA(cudaEventRecordWithFlags(pl->pev[id][1], pl->stream,
                                     pl->capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
    pl->pending[id] = true;
}
inline void prof_collect(se_plan *pl) {
    if (!pl->prof) return;
    for (int id = 0; id < SE_K_COUNT; ++id) {
        if (!pl->pending[id]) continue;
        SE_CUDA(cudaEventSynchronize(pl->pev[id][1]));
        float ms = 0;
        SE_CUDA(cudaEventElapsedTime(&ms, pl->pev[id][0], pl->pev[id][1]));
        pl->pms[id] += ms;
        pl->pcount[id] += 1;
        pl->pending[id] = false;
    }
}

// launch helpers (defined in the .cu files)
void realspace_pair_count(se_plan *pl, const double *pos, const double *q, int64_t N, long long *pairs);
void spread_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *grid,
                int rank, int world);
void gather_run(se_plan *pl, const double *grid, const double *pos, int64_t N, double *phi,
                int accumulate, int rank, int world, bool rebin);
void kspace_run(se_plan *pl, double *grid, int use_kernel, double *timings);
void realspace_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi,
                   int add_self, int rank, int world);
void grad_gather_run(se_plan *pl, const double *grid, const double *pos, int64_t N, double *E, int accumulate);
void zslab_geometry(se_plan *pl, int world, int rank, int64_t *out);
void zslab_forward(se_plan *pl, int world, int rank, const double *zslab, double *spec);
void zslab_rows(se_plan *pl, int world, int rank, double *recv);
void zslab_inverse(se_plan *pl, int world, int rank, const double *spec, double *zslab);
void realspace_domain_run(se_plan *pl, const double *pos, const double *q, int64_t n_local, int64_t n_own, int ncols,
                          int col_lo, int col_hi, double *phi, int add_self);
void realspace_field_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *E,
                         int rank, int world);
void d0_kernel_prepare(se_plan *pl, double *t_precompute);
void kspace_field_run(se_plan *pl, double *grid, double *g3);
void slab_geometry(se_plan *pl, int world, int64_t *nx, int64_t *nky, int64_t *nkz);
void slab_forward(se_plan *pl, int world, const double *slab, double *send);
void slab_xpass(se_plan *pl, int world, int rank, double *recv);
void slab_inverse(se_plan *pl, int world, const double *back, double *slab);
void plan_release_device(se_plan *pl);

// binning (se_sort.cu)
void binning_reserve(se_plan *pl, Binning &b, int64_t N, int nbins, int chunk, int extra_bits = 0);
void binning_sort(se_plan *pl, Binning &b, const double *pos, const double *q, int64_t N, int nbins, int chunk,
                  int extra_bits = 0, int64_t rlo = 0, int ubin_lo = 0, int ubin_hi = -1);
int64_t binning_max_units(const Binning &b, int64_t N, int nbins, int chunk);

// shared device helpers ---------------------------------------------------
// A coordinate as the binning kernels use it.  Valid input (x in [0, L)) is
// returned unchanged.  The fused total-potential call reports a coordinate
// outside the box (core.py:65-77) only AFTER its device work, without a host
// round trip up front; until then such a coordinate (NaN included) is replaced
// by a pseudo-random point of the box derived from its index, identically in
// the key and the record kernels, so every later kernel indexes in range and
// no bin piles up.  The results of such a call are discarded by the error.
#ifdef __CUDACC__
__device__ __forceinline__ double sane_coord(double x, double L, long long i, int ax) {
    if (x >= 0.0 && x < L) return x;
    const unsigned h = (unsigned)(3 * i + ax) * 2654435761u;
    return L * ((double)(h >> 8) * (1.0 / 16777216.0));
}
#endif
struct WinParams {
    int window;
    int P;
    double h, w, shape;
    double peak;   // gaussian: m / (w sqrt(2 pi))
    double i0b;    // kb: I0(beta)
};

__host__ __device__ inline WinParams make_win(const se_params_t &p, double h) {
    WinParams wp;
    wp.window = p.window;
    wp.P = p.P;
    wp.h = h;
    wp.w = 0.5 * p.P * h;
    wp.shape = p.shape;
    wp.peak = p.shape / (wp.w * 2.5066282746310002);  // sqrt(2 pi)
    wp.i0b = 1.0;
    return wp;
}

}  // namespace se
