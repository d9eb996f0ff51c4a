// k-space stage of the SE pipeline on cuFFT plus fused multiplier kernels.
//
//  D=3  aft_forward/scale/aft_inverse (aft.py:203-206, sekspace.py:198-206,
//       aft.py:237-238): real-to-complex M^3 FFT, one pass multiplying by
//       4 pi e^{-k^2/4xi^2} / (k^2 w^2) (0 at k=0), complex-to-real FFT.
//  D=2,1 adaptive FFT (aft.py:155-265, sekspace.py:217-254): the periodic
//       transform is real-to-complex, so only the half plane of periodic
//       modes is carried (the free-axis operator commutes with conjugation);
//       rows/planes of the zero block (padded to g0), the I block (padded to
//       gs) and the J block (unpadded Mt) are transformed as three batched
//       cuFFT calls, scaled by one fused kernel per block, inverted,
//       restricted to Mt and merged back before the inverse periodic
//       transform.
//  D=0  precomputed truncated kernel on the 2x padded grid
//       (sekspace.py:257-337), including the one-time precompute of the
//       kernel table on the device (fine g0^3 grid, inverse transform, clip,
//       forward transform), or the globally upsampled path
//       (use_kernel = False, sekspace.py:208-215).
#include <cuda_runtime.h>

#include "se_common.h"

namespace se {

typedef double2 cplx;

// ------------------------------------------------------------- tables
static void upload(DevBuf &b, const std::vector<double> &v) {
    b.ensure(sizeof(double) * (v.size() ? v.size() : 1));
    SE_CUDA(cudaMemcpy(b.ptr, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice));
}

// sekspace.py:181-185 (_window_table with its underflow guard)
static void make_table(se_plan *pl, ModeTable &t, int n, bool half) {
    std::vector<double> k;
    if (half) {  // 2 pi rfftfreq(n, d=h)
        int nh = n / 2 + 1;
        k.resize(nh);
        double val = 1.0 / (n * pl->g.h);
        for (int j = 0; j < nh; ++j) k[j] = 2.0 * M_PI * (j * val);
    } else {
        k = wavenumbers(n, pl->g.h);
    }
    std::vector<double> w = window_fourier(pl->p.window, pl->p.P, pl->g.h, pl->p.shape, k);
    double mn = 1e300;
    for (double v : w) mn = std::fmin(mn, std::fabs(v));
    if (mn < 1e-30) fail(SE_ENUMERIC, "window transform underflow: P/M misconfigured");
    t.n = (int)k.size();
    upload(t.k, k);
    upload(t.what, w);
}

// ------------------------------------------------------------- helpers
__device__ __forceinline__ double mollify(double k2, double xi) { return exp(-k2 / (4.0 * xi * xi)); }

// greens.py:48-85 on the device (zero periodic-mode block)
__device__ double greens_zero_dev(int D, double R, double kappa) {
    kappa = fabs(kappa);
    double t = R * kappa;
    if (t < 1e-2) {
        double z = t * t;
        if (D == 0) return R * R * (0.5 - z / 24.0 + z * z / 720.0 - z * z * z / 40320.0 + z * z * z * z / 3628800.0);
        if (D == 1) {
            double lr = log(R);
            return R * R * ((0.25 - 0.5 * lr) - z * (1.0 / 64.0 - lr / 16.0) + z * z * (1.0 / 2304.0 - lr / 384.0) -
                            z * z * z * (1.0 / 147456.0 - lr / 18432.0) +
                            z * z * z * z * (1.0 / 14745600.0 - lr / 1474560.0));
        }
        return R * R * (-0.5 + z / 8.0 - z * z / 144.0 + z * z * z / 5760.0 - z * z * z * z / 403200.0);
    }
    if (D == 0) return R * R * (1.0 - cos(t)) / (t * t);
    if (D == 1) return (1.0 - j0(t)) / (kappa * kappa) - (R * log(R)) * j1(t) / kappa;
    return R * R * (1.0 - cos(t) - t * sin(t)) / (t * t);
}

__global__ void scale_d3_kernel(cplx *__restrict__ F, int M, const double *__restrict__ k, const double *__restrict__ w,
                                double xi, double norm) {
    const int nh = M / 2 + 1;
    int64_t total = (int64_t)M * M * nh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int iz = (int)(i % nh);
        int64_t r = i / nh;
        int iy = (int)(r % M), ix = (int)(r / M);
        double k2 = k[ix] * k[ix] + k[iy] * k[iy] + k[iz] * k[iz];
        double W = w[ix] * w[iy] * w[iz];
        double fac = k2 > 0.0 ? 4.0 * M_PI * mollify(k2, xi) * (1.0 / k2) / (W * W) * norm : 0.0;
        cplx v = F[i];
        F[i] = make_double2(v.x * fac, v.y * fac);
    }
}

__global__ void pad_real_kernel(const double *__restrict__ src, int s0, int s1, int s2, double *__restrict__ dst, int d0,
                                int d1, int d2) {
    int64_t total = (int64_t)d0 * d1 * d2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int z = (int)(i % d2);
        int64_t r = i / d2;
        int y = (int)(r % d1), x = (int)(r / d1);
        dst[i] = (x < s0 && y < s1 && z < s2) ? src[((int64_t)x * s1 + y) * s2 + z] : 0.0;
    }
}

__global__ void restrict_real_kernel(const double *__restrict__ src, int d1, int d2, double *__restrict__ dst, int s0,
                                     int s1, int s2, double scale) {
    int64_t total = (int64_t)s0 * s1 * s2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int z = (int)(i % s2);
        int64_t r = i / s2;
        int y = (int)(r % s1), x = (int)(r / s1);
        dst[i] = src[((int64_t)x * d1 + y) * d2 + z] * scale;
    }
}

// D=0 kernel path: F *= ghat * 4 pi * af[x] * af[y] * ah[z] / n^3  (sekspace.py:319-326)
__global__ void scale_d0k_kernel(cplx *__restrict__ F, int n, const double *__restrict__ ghat,
                                 const double *__restrict__ af, const double *__restrict__ ah, double norm) {
    const int nh = n / 2 + 1;
    int64_t total = (int64_t)n * n * nh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int iz = (int)(i % nh);
        int64_t r = i / nh;
        int iy = (int)(r % n), ix = (int)(r / n);
        double fac = ghat[i] * (4.0 * M_PI * af[ix]) * af[iy] * ah[iz] * norm;
        cplx v = F[i];
        F[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// D=0 full upsampling: F *= 4 pi e^{-k^2/4xi^2} G0(|k|) / W^2 / g^3  (sekspace.py:208-215)
__global__ void scale_d0f_kernel(cplx *__restrict__ F, int g, const double *__restrict__ k, const double *__restrict__ w,
                                 double xi, double R, double norm) {
    const int gh = g / 2 + 1;
    int64_t total = (int64_t)g * g * gh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int iz = (int)(i % gh);
        int64_t r = i / gh;
        int iy = (int)(r % g), ix = (int)(r / g);
        double k2 = k[ix] * k[ix] + k[iy] * k[iy] + k[iz] * k[iz];
        double W = w[ix] * w[iy] * w[iz];
        double fac = 4.0 * M_PI * mollify(k2, xi) * greens_zero_dev(0, R, sqrt(k2)) / (W * W) * norm;
        cplx v = F[i];
        F[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// half spectrum of G0 on the fine grid (imaginary part zero)
__global__ void ghat_fine_kernel(cplx *__restrict__ out, int g, const double *__restrict__ k, double R) {
    const int gh = g / 2 + 1;
    int64_t total = (int64_t)g * g * gh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int iz = (int)(i % gh);
        int64_t r = i / gh;
        int iy = (int)(r % g), ix = (int)(r / g);
        double k2 = k[ix] * k[ix] + k[iy] * k[iy] + k[iz] * k[iz];
        out[i] = make_double2(greens_zero_dev(0, R, sqrt(k2)), 0.0);
    }
}

// clip cube [0,half) U [g-half,g) per axis of the fine real kernel (sekspace.py:291-293)
__global__ void clip_cube_kernel(const double *__restrict__ fine, int g, double *__restrict__ cube, int n, double scale) {
    const int half = n / 2;
    int64_t total = (int64_t)n * n * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int z = (int)(i % n);
        int64_t r = i / n;
        int y = (int)(r % n), x = (int)(r / n);
        int sx = x < half ? x : g - n + x, sy = y < half ? y : g - n + y, sz = z < half ? z : g - n + z;
        cube[i] = fine[((int64_t)sx * g + sy) * g + sz] * scale;
    }
}

__global__ void take_real_kernel(const cplx *__restrict__ in, double *__restrict__ out, int64_t total,
                                 unsigned long long *__restrict__ mx) {
    double mre = 0.0, mim = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        cplx v = in[i];
        out[i] = v.x;
        mre = fmax(mre, fabs(v.x));
        mim = fmax(mim, fabs(v.y));
    }
    for (int o = 16; o > 0; o >>= 1) {
        mre = fmax(mre, __shfl_xor_sync(0xffffffffu, mre, o));
        mim = fmax(mim, __shfl_xor_sync(0xffffffffu, mim, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(mx, (unsigned long long)__double_as_longlong(mre));
        atomicMax(mx + 1, (unsigned long long)__double_as_longlong(mim));
    }
}

// ------------------------------------------------ mixed periodicity (AFT)
// pack rows/planes of Hk into a zero-padded batch: dst[r][...] (glen^nfree)
__global__ void pack_kernel(const cplx *__restrict__ Hk, int Mt, int nfree, const int *__restrict__ rows, int nrows,
                            cplx *__restrict__ dst, int glen) {
    int64_t per = nfree == 1 ? glen : (int64_t)glen * glen;
    int64_t src_per = nfree == 1 ? Mt : (int64_t)Mt * Mt;
    int64_t total = per * nrows;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int r = (int)(i / per);
        int64_t e = i - (int64_t)r * per;
        int row = rows ? rows[r] : 0;
        cplx v = make_double2(0.0, 0.0);
        if (nfree == 1) {
            if (e < Mt) v = Hk[(int64_t)row * src_per + e];
        } else {
            int y = (int)(e / glen), z = (int)(e - (int64_t)y * glen);
            if (y < Mt && z < Mt) v = Hk[(int64_t)row * src_per + (int64_t)y * Mt + z];
        }
        dst[i] = v;
    }
}

__global__ void unpack_kernel(const cplx *__restrict__ src, int glen, int nfree, const int *__restrict__ rows, int nrows,
                              cplx *__restrict__ Hk, int Mt) {
    int64_t dper = nfree == 1 ? Mt : (int64_t)Mt * Mt;
    int64_t sper = nfree == 1 ? glen : (int64_t)glen * glen;
    int64_t total = dper * nrows;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int r = (int)(i / dper);
        int64_t e = i - (int64_t)r * dper;
        int row = rows ? rows[r] : 0;
        int64_t s;
        if (nfree == 1) {
            s = e;
        } else {
            int y = (int)(e / Mt), z = (int)(e - (int64_t)y * Mt);
            s = (int64_t)y * glen + z;
        }
        Hk[(int64_t)row * dper + e] = src[(int64_t)r * sper + s];
    }
}

struct MixArgs {
    int D, M, nI, half;  // half = M/2+1 (number of carried modes along the halved periodic axis)
    double xi, R;
    const double *kp, *wp;  // periodic mode table (length M)
    int row0 = 0, nrows = -1;  // a chunk of the periodic-mode rows (multi-GPU); nrows < 0: all rows
};

__device__ __forceinline__ int absmode(int i, int M) { return i < M / 2 ? i : M - i; }

// J-block multiplier applied to every row/plane of Hk whose max-norm mode
// exceeds nI (sekspace.py:234-254).  Rows of the zero/I blocks are skipped
// (they are replaced by the unpack of their padded transforms).
// D=2: Hk layout [ix][iy<half][z] (rows of Mt); D=1: [ix<half][y][z].
__global__ void scale_mixJ_kernel(cplx *__restrict__ Hk, MixArgs a, int Mt, const double *__restrict__ kf,
                                  const double *__restrict__ wf, double norm) {
    const int nfree = 3 - a.D;
    int64_t per = nfree == 1 ? Mt : (int64_t)Mt * Mt;
    int64_t rowsN = a.nrows >= 0 ? a.nrows : (a.D == 2 ? (int64_t)a.M * a.half : a.half);
    int64_t total = rowsN * per;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lrow = i / per;
        const int64_t e = i - lrow * per;
        const int64_t row = lrow + a.row0;
        double kr2, wr;
        int mu;
        if (a.D == 2) {
            int ix = (int)(row / a.half), iy = (int)(row - (int64_t)ix * a.half);
            mu = max(absmode(ix, a.M), absmode(iy, a.M));
            kr2 = a.kp[ix] * a.kp[ix] + a.kp[iy] * a.kp[iy];
            wr = a.wp[ix] * a.wp[iy];
        } else {
            int ix = (int)row;
            mu = absmode(ix, a.M);
            kr2 = a.kp[ix] * a.kp[ix];
            wr = a.wp[ix];
        }
        if (mu <= a.nI) continue;
        double k2, W;
        if (nfree == 1) {
            k2 = kr2 + kf[e] * kf[e];
            W = wr * wf[e];
        } else {
            int y = (int)(e / Mt), z = (int)(e - (int64_t)y * Mt);
            k2 = kr2 + kf[y] * kf[y] + kf[z] * kf[z];
            W = wr * (wf[y] * wf[z]);
        }
        double fac = 4.0 * M_PI * mollify(k2, a.xi) / (k2 * (W * W)) * norm;
        cplx v = Hk[i];
        Hk[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// I-block multiplier on the packed, padded rows (glen = gs).
__global__ void scale_mixI_kernel(cplx *__restrict__ B, MixArgs a, const int *__restrict__ rows, int nrows, int glen,
                                  const double *__restrict__ kf, const double *__restrict__ wf, double norm) {
    const int nfree = 3 - a.D;
    int64_t per = nfree == 1 ? glen : (int64_t)glen * glen;
    int64_t total = per * nrows;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int r = (int)(i / per);
        int64_t e = i - (int64_t)r * per;
        int row = rows[r] + a.row0;  // rows[] index the (chunk's) rows; modes are global
        double kr2, wr;
        if (a.D == 2) {
            int ix = row / a.half, iy = row - ix * a.half;
            kr2 = a.kp[ix] * a.kp[ix] + a.kp[iy] * a.kp[iy];
            wr = a.wp[ix] * a.wp[iy];
        } else {
            kr2 = a.kp[row] * a.kp[row];
            wr = a.wp[row];
        }
        double k2, W;
        if (nfree == 1) {
            k2 = kr2 + kf[e] * kf[e];
            W = wr * wf[e];
        } else {
            int y = (int)(e / glen), z = (int)(e - (int64_t)y * glen);
            k2 = kr2 + kf[y] * kf[y] + kf[z] * kf[z];
            W = wr * (wf[y] * wf[z]);
        }
        double fac = 4.0 * M_PI * mollify(k2, a.xi) / (k2 * (W * W)) * norm;
        cplx v = B[i];
        B[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// zero block multiplier (sekspace.py:221-232), glen = g0
__global__ void scale_mix0_kernel(cplx *__restrict__ Z, MixArgs a, int glen, const double *__restrict__ kf,
                                  const double *__restrict__ wf, double norm) {
    const int nfree = 3 - a.D;
    int64_t total = nfree == 1 ? glen : (int64_t)glen * glen;
    double wp0 = a.D == 2 ? a.wp[0] * a.wp[0] : a.wp[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        double kap2, wfree;
        if (nfree == 1) {
            kap2 = kf[i] * kf[i];
            wfree = wf[i];
        } else {
            int y = (int)(i / glen), z = (int)(i - (int64_t)y * glen);
            kap2 = kf[y] * kf[y] + kf[z] * kf[z];
            wfree = wf[y] * wf[z];
        }
        double W = wp0 * wfree;
        double fac = 4.0 * M_PI * mollify(kap2, a.xi) * greens_zero_dev(a.D, a.R, sqrt(kap2)) / (W * W) * norm;
        cplx v = Z[i];
        Z[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// ------------------------------------------------------------- launch utils
static unsigned grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return (unsigned)b;
}

#define LAUNCH(kern, total, ...)                                                   \
    do {                                                                           \
        kern<<<grid_for(total), 256, 0, pl->stream>>>(__VA_ARGS__);                \
        SE_LAUNCH_CHECK();                                                         \
        pl->launches += 1;                                                         \
    } while (0)

struct StageTimer {
    se_plan *pl;
    bool on;
    cudaEvent_t ev[8];
    int n = 0;
    StageTimer(se_plan *p, bool enabled) : pl(p), on(enabled) {
        if (on)
            for (auto &e : ev) SE_CUDA(cudaEventCreate(&e));
    }
    void mark() {
        if (on) SE_CUDA(cudaEventRecord(ev[n++], pl->stream));
    }
    double secs(int a, int b) {
        float ms = 0;
        SE_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
        return ms * 1e-3;
    }
    ~StageTimer() {
        if (on)
            for (auto &e : ev) cudaEventDestroy(e);
    }
};

// ------------------------------------------------------------- plans
static void ensure_tables(se_plan *pl) {
    if (pl->kspace_ready) return;
    const int D = pl->D;
    const se_grid_t &g = pl->g;
    if (D == 3) {
        make_table(pl, pl->tM, g.M, false);
    } else if (D == 0) {
        make_table(pl, pl->tg0, g.g0, false);
    } else {
        make_table(pl, pl->tM, g.M, false);
        make_table(pl, pl->tg0, g.g0, false);
        make_table(pl, pl->tMt, g.Mt, false);
        if (pl->nI_rows >= 0) make_table(pl, pl->tgs, g.gs, false);
        // I rows of the half plane
        std::vector<int> rows;
        const int M = g.M, half = M / 2 + 1;
        std::vector<int> m = signed_modes(M);
        if (D == 2) {
            for (int ix = 0; ix < M; ++ix)
                for (int iy = 0; iy < half; ++iy) {
                    int mu = std::max(std::abs(m[ix]), std::abs(m[iy]));
                    if (mu >= 1 && mu <= pl->p.nI) rows.push_back(ix * half + iy);
                }
        } else {
            for (int ix = 0; ix < half; ++ix) {
                int mu = std::abs(m[ix]);
                if (mu >= 1 && mu <= pl->p.nI) rows.push_back(ix);
            }
        }
        pl->nI_rows = (int)rows.size();
        pl->rows_I.ensure(sizeof(int) * (rows.size() + 1));
        if (!rows.empty())
            SE_CUDA(cudaMemcpy(pl->rows_I.ptr, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    }
    pl->kspace_ready = true;
}

static void make_ffts(se_plan *pl) {
    if (pl->fft_made) return;
    const se_grid_t &g = pl->g;
    const int D = pl->D, M = g.M, Mt = g.Mt;
    if (D == 3) {
        SE_CUFFT(cufftPlan3d(&pl->fft_fwd, M, M, M, CUFFT_D2Z));
        SE_CUFFT(cufftPlan3d(&pl->fft_inv, M, M, M, CUFFT_Z2D));
        pl->spec.ensure(sizeof(cplx) * (size_t)M * M * (M / 2 + 1));
    } else if (D == 2) {
        const int half = M / 2 + 1;
        int n[2] = {M, M}, rin[2] = {M, M}, cout[2] = {M, half};
        SE_CUFFT(cufftPlanMany(&pl->fft_fwd, 2, n, rin, Mt, 1, cout, Mt, 1, CUFFT_D2Z, Mt));
        SE_CUFFT(cufftPlanMany(&pl->fft_inv, 2, n, cout, Mt, 1, rin, Mt, 1, CUFFT_Z2D, Mt));
        int nJ[1] = {Mt}, nI1[1] = {g.gs}, n0[1] = {g.g0};
        SE_CUFFT(cufftPlanMany(&pl->fft_rowJ, 1, nJ, nullptr, 1, Mt, nullptr, 1, Mt, CUFFT_Z2Z, M * half));
        if (pl->nI_rows > 0)
            SE_CUFFT(cufftPlanMany(&pl->fft_rowI, 1, nI1, nullptr, 1, g.gs, nullptr, 1, g.gs, CUFFT_Z2Z, pl->nI_rows));
        SE_CUFFT(cufftPlanMany(&pl->fft_row0, 1, n0, nullptr, 1, g.g0, nullptr, 1, g.g0, CUFFT_Z2Z, 1));
        pl->spec.ensure(sizeof(cplx) * (size_t)M * half * Mt);
        pl->spec2.ensure(sizeof(cplx) * (size_t)g.g0);
        pl->spec3.ensure(sizeof(cplx) * (size_t)(pl->nI_rows ? pl->nI_rows : 1) * g.gs);
    } else if (D == 1) {
        const int half = M / 2 + 1;
        int n[1] = {M}, rin[1] = {M}, cout[1] = {half};
        SE_CUFFT(cufftPlanMany(&pl->fft_fwd, 1, n, rin, Mt * Mt, 1, cout, Mt * Mt, 1, CUFFT_D2Z, Mt * Mt));
        SE_CUFFT(cufftPlanMany(&pl->fft_inv, 1, n, cout, Mt * Mt, 1, rin, Mt * Mt, 1, CUFFT_Z2D, Mt * Mt));
        int nJ[2] = {Mt, Mt}, nI2[2] = {g.gs, g.gs}, n0[2] = {g.g0, g.g0};
        SE_CUFFT(cufftPlanMany(&pl->fft_rowJ, 2, nJ, nullptr, 1, Mt * Mt, nullptr, 1, Mt * Mt, CUFFT_Z2Z, half));
        if (pl->nI_rows > 0)
            SE_CUFFT(cufftPlanMany(&pl->fft_rowI, 2, nI2, nullptr, 1, g.gs * g.gs, nullptr, 1, g.gs * g.gs, CUFFT_Z2Z,
                                   pl->nI_rows));
        SE_CUFFT(cufftPlanMany(&pl->fft_row0, 2, n0, nullptr, 1, g.g0 * g.g0, nullptr, 1, g.g0 * g.g0, CUFFT_Z2Z, 1));
        pl->spec.ensure(sizeof(cplx) * (size_t)half * Mt * Mt);
        pl->spec2.ensure(sizeof(cplx) * (size_t)g.g0 * g.g0);
        pl->spec3.ensure(sizeof(cplx) * (size_t)(pl->nI_rows ? pl->nI_rows : 1) * g.gs * g.gs);
    }
    pl->fft_made = true;
}

static void set_streams(se_plan *pl, std::initializer_list<cufftHandle> hs) {
    for (cufftHandle h : hs)
        if (h) SE_CUFFT(cufftSetStream(h, pl->stream));
}

// ------------------------------------------------------------- D = 0 kernel
void d0_kernel_prepare(se_plan *pl, double *t_pre) {
    if (pl->d0_ready) {
        if (t_pre) *t_pre = 0.0;
        return;
    }
    StageTimer tm(pl, t_pre != nullptr);
    tm.mark();
    const se_grid_t &g = pl->g;
    D0Geom d = d0_geometry(g.L, g.M, g.P, pl->p.s0, pl->p.rc, true);
    pl->nconv = d.nconv;
    pl->kg0 = d.g0;
    pl->kR = d.R;
    const int gf = d.g0, n = d.nconv, nh = n / 2 + 1;
    // fine grid wavenumbers (window-independent)
    std::vector<double> kf = wavenumbers(gf, g.h);
    DevBuf dk;
    upload(dk, kf);
    DevBuf half, fine;
    half.ensure(sizeof(cplx) * (size_t)gf * gf * (gf / 2 + 1));
    fine.ensure(sizeof(double) * (size_t)gf * gf * gf);
    LAUNCH(ghat_fine_kernel, (int64_t)gf * gf * (gf / 2 + 1), half.as<cplx>(), gf, dk.as<double>(), d.R);
    cufftHandle hinv = 0, hfwd = 0;
    SE_CUFFT(cufftPlan3d(&hinv, gf, gf, gf, CUFFT_Z2D));
    SE_CUFFT(cufftSetStream(hinv, pl->stream));
    SE_CUFFT(cufftExecZ2D(hinv, half.as<cplx>(), fine.as<double>()));
    cufftDestroy(hinv);
    half.release();
    DevBuf cube, cspec;
    cube.ensure(sizeof(double) * (size_t)n * n * n);
    // numpy ifftn normalisation 1/g^3; the reference's /h^3 and h^3 cancel
    double scale = 1.0 / ((double)gf * gf * gf);
    LAUNCH(clip_cube_kernel, (int64_t)n * n * n, fine.as<double>(), gf, cube.as<double>(), n, scale);
    fine.release();
    cspec.ensure(sizeof(cplx) * (size_t)n * n * nh);
    SE_CUFFT(cufftPlan3d(&hfwd, n, n, n, CUFFT_D2Z));
    SE_CUFFT(cufftSetStream(hfwd, pl->stream));
    SE_CUFFT(cufftExecD2Z(hfwd, cube.as<double>(), cspec.as<cplx>()));
    cufftDestroy(hfwd);
    cube.release();
    pl->ghat.ensure(sizeof(double) * (size_t)n * n * nh);
    DevBuf mx;
    mx.ensure(2 * sizeof(unsigned long long));
    SE_CUDA(cudaMemsetAsync(mx.ptr, 0, 2 * sizeof(unsigned long long), pl->stream));
    LAUNCH(take_real_kernel, (int64_t)n * n * nh, cspec.as<cplx>(), pl->ghat.as<double>(), (int64_t)n * n * nh,
           mx.as<unsigned long long>());
    unsigned long long hm[2];
    SE_CUDA(cudaMemcpyAsync(hm, mx.ptr, sizeof(hm), cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
    cspec.release();
    double mre, mim;
    memcpy(&mre, &hm[0], 8);
    memcpy(&mim, &hm[1], 8);
    if (!(mim < 1e-13 * mre)) fail(SE_ENUMERIC, "truncated kernel transform must be real");
    // per-axis factors a = e^{-k^2/4xi^2} / w^2 on the full and half mode sets
    make_table(pl, pl->tNc, n, false);
    make_table(pl, pl->tNh, n, true);
    auto afac = [&](ModeTable &t) {
        std::vector<double> k(t.n), w(t.n), a(t.n);
        SE_CUDA(cudaMemcpy(k.data(), t.k.ptr, sizeof(double) * t.n, cudaMemcpyDeviceToHost));
        SE_CUDA(cudaMemcpy(w.data(), t.what.ptr, sizeof(double) * t.n, cudaMemcpyDeviceToHost));
        const double xi = pl->p.xi;
        for (int i = 0; i < t.n; ++i) a[i] = std::exp(-(k[i] * k[i]) / (4.0 * xi * xi)) / (w[i] * w[i]);
        upload(t.what, a);  // reuse the slot: holds a(k) from here on
    };
    afac(pl->tNc);
    afac(pl->tNh);
    SE_CUFFT(cufftPlan3d(&pl->fft_c_fwd, n, n, n, CUFFT_D2Z));
    SE_CUFFT(cufftPlan3d(&pl->fft_c_inv, n, n, n, CUFFT_Z2D));
    pl->d0_fft_made = true;
    pl->d0_ready = true;
    tm.mark();
    if (t_pre) {
        SE_CUDA(cudaStreamSynchronize(pl->stream));
        *t_pre = tm.secs(0, 1);
    }
}

// ------------------------------------------------------------- driver
void kspace_run(se_plan *pl, double *grid, int use_kernel, double *timings) {
    const int D = pl->D;
    const se_grid_t &g = pl->g;
    if (timings) timings[SE_T_PRECOMPUTE] = 0.0;
    ensure_tables(pl);
    StageTimer tm(pl, timings != nullptr);
    if (D == 0 && use_kernel) {
        d0_kernel_prepare(pl, timings ? &timings[SE_T_PRECOMPUTE] : nullptr);
        const int n = pl->nconv, nh = n / 2 + 1, Mt = g.Mt;
        pl->grid_tmp.ensure(sizeof(double) * (size_t)n * n * n);
        pl->spec.ensure(sizeof(cplx) * (size_t)n * n * nh);
        set_streams(pl, {pl->fft_c_fwd, pl->fft_c_inv});
        tm.mark();
        LAUNCH(pad_real_kernel, (int64_t)n * n * n, grid, Mt, Mt, Mt, pl->grid_tmp.as<double>(), n, n, n);
        SE_CUFFT(cufftExecD2Z(pl->fft_c_fwd, pl->grid_tmp.as<double>(), pl->spec.as<cplx>()));
        tm.mark();
        LAUNCH(scale_d0k_kernel, (int64_t)n * n * nh, pl->spec.as<cplx>(), n, pl->ghat.as<double>(),
               pl->tNc.what.as<double>(), pl->tNh.what.as<double>(), 1.0 / ((double)n * n * n));
        tm.mark();
        SE_CUFFT(cufftExecZ2D(pl->fft_c_inv, pl->spec.as<cplx>(), pl->grid_tmp.as<double>()));
        LAUNCH(restrict_real_kernel, (int64_t)Mt * Mt * Mt, pl->grid_tmp.as<double>(), n, n, grid, Mt, Mt, Mt, 1.0);
        tm.mark();
    } else if (D == 0) {
        const int gf = g.g0, gh = gf / 2 + 1, Mt = g.Mt;
        if (!pl->d0full_fft_made) {
            SE_CUFFT(cufftPlan3d(&pl->fft_f_fwd, gf, gf, gf, CUFFT_D2Z));
            SE_CUFFT(cufftPlan3d(&pl->fft_f_inv, gf, gf, gf, CUFFT_Z2D));
            pl->d0full_fft_made = true;
        }
        pl->grid_tmp.ensure(sizeof(double) * (size_t)gf * gf * gf);
        pl->spec.ensure(sizeof(cplx) * (size_t)gf * gf * gh);
        set_streams(pl, {pl->fft_f_fwd, pl->fft_f_inv});
        tm.mark();
        LAUNCH(pad_real_kernel, (int64_t)gf * gf * gf, grid, Mt, Mt, Mt, pl->grid_tmp.as<double>(), gf, gf, gf);
        SE_CUFFT(cufftExecD2Z(pl->fft_f_fwd, pl->grid_tmp.as<double>(), pl->spec.as<cplx>()));
        tm.mark();
        LAUNCH(scale_d0f_kernel, (int64_t)gf * gf * gh, pl->spec.as<cplx>(), gf, pl->tg0.k.as<double>(),
               pl->tg0.what.as<double>(), pl->p.xi, g.R, 1.0 / ((double)gf * gf * gf));
        tm.mark();
        SE_CUFFT(cufftExecZ2D(pl->fft_f_inv, pl->spec.as<cplx>(), pl->grid_tmp.as<double>()));
        LAUNCH(restrict_real_kernel, (int64_t)Mt * Mt * Mt, pl->grid_tmp.as<double>(), gf, gf, grid, Mt, Mt, Mt, 1.0);
        tm.mark();
    } else if (D == 3) {
        make_ffts(pl);
        set_streams(pl, {pl->fft_fwd, pl->fft_inv});
        const int M = g.M;
        tm.mark();
        SE_CUFFT(cufftExecD2Z(pl->fft_fwd, grid, pl->spec.as<cplx>()));
        tm.mark();
        LAUNCH(scale_d3_kernel, (int64_t)M * M * (M / 2 + 1), pl->spec.as<cplx>(), M, pl->tM.k.as<double>(),
               pl->tM.what.as<double>(), pl->p.xi, 1.0 / ((double)M * M * M));
        tm.mark();
        SE_CUFFT(cufftExecZ2D(pl->fft_inv, pl->spec.as<cplx>(), grid));
        tm.mark();
    } else {
        if (g.Mt % 2) fail(SE_EINVAL, "free-axis grid size must be even");
        make_ffts(pl);
        set_streams(pl, {pl->fft_fwd, pl->fft_inv, pl->fft_rowJ, pl->fft_rowI, pl->fft_row0});
        const int M = g.M, Mt = g.Mt, half = M / 2 + 1, nfree = 3 - D;
        const int nI = pl->nI_rows;
        cplx *Hk = pl->spec.as<cplx>(), *Z = pl->spec2.as<cplx>(), *B = pl->spec3.as<cplx>();
        const int *rows = pl->rows_I.as<int>();
        MixArgs ma{D, M, pl->p.nI, half, pl->p.xi, g.R, pl->tM.k.as<double>(), pl->tM.what.as<double>()};
        const double perN = D == 2 ? (double)M * M : (double)M;
        auto pw = [&](int n) { return nfree == 1 ? (double)n : (double)n * n; };
        tm.mark();
        SE_CUFFT(cufftExecD2Z(pl->fft_fwd, grid, Hk));
        LAUNCH(pack_kernel, (int64_t)pw(g.g0), Hk, Mt, nfree, nullptr, 1, Z, g.g0);
        if (nI) LAUNCH(pack_kernel, (int64_t)pw(g.gs) * nI, Hk, Mt, nfree, rows, nI, B, g.gs);
        SE_CUFFT(cufftExecZ2Z(pl->fft_rowJ, Hk, Hk, CUFFT_FORWARD));
        if (nI) SE_CUFFT(cufftExecZ2Z(pl->fft_rowI, B, B, CUFFT_FORWARD));
        SE_CUFFT(cufftExecZ2Z(pl->fft_row0, Z, Z, CUFFT_FORWARD));
        tm.mark();
        int64_t rowsN = D == 2 ? (int64_t)M * half : half;
        LAUNCH(scale_mixJ_kernel, rowsN * (int64_t)pw(Mt), Hk, ma, Mt, pl->tMt.k.as<double>(),
               pl->tMt.what.as<double>(), 1.0 / (pw(Mt) * perN));
        if (nI)
            LAUNCH(scale_mixI_kernel, (int64_t)pw(g.gs) * nI, B, ma, rows, nI, g.gs, pl->tgs.k.as<double>(),
                   pl->tgs.what.as<double>(), 1.0 / (pw(g.gs) * perN));
        LAUNCH(scale_mix0_kernel, (int64_t)pw(g.g0), Z, ma, g.g0, pl->tg0.k.as<double>(), pl->tg0.what.as<double>(),
               1.0 / (pw(g.g0) * perN));
        tm.mark();
        SE_CUFFT(cufftExecZ2Z(pl->fft_rowJ, Hk, Hk, CUFFT_INVERSE));
        if (nI) SE_CUFFT(cufftExecZ2Z(pl->fft_rowI, B, B, CUFFT_INVERSE));
        SE_CUFFT(cufftExecZ2Z(pl->fft_row0, Z, Z, CUFFT_INVERSE));
        if (nI) LAUNCH(unpack_kernel, (int64_t)pw(Mt) * nI, B, g.gs, nfree, rows, nI, Hk, Mt);
        LAUNCH(unpack_kernel, (int64_t)pw(Mt), Z, g.g0, nfree, nullptr, 1, Hk, Mt);
        SE_CUFFT(cufftExecZ2D(pl->fft_inv, Hk, grid));
        tm.mark();
    }
    if (timings) {
        SE_CUDA(cudaStreamSynchronize(pl->stream));
        timings[SE_T_AFT] = tm.secs(0, 1);
        timings[SE_T_SCALE] = tm.secs(1, 2);
        timings[SE_T_AIFT] = tm.secs(2, 3);
    }
}

// --------------------------------------------------- slab-decomposed D = 3
// The k-space stage of D = 3 over `world` ranks: rank r owns the
// x-slab of nx = M / world planes (the C-order grid's contiguous block r, as
// a reduce-scatter leaves it).  Forward: 2-D R2C over (y, z) of the slab's
// planes, packed into (world, nx, nky, nkz) blocks (block s = this rank's
// planes x ky-chunk s) for an all-to-all; after it each rank holds all kx
// for its ky-chunk, (M, nky, nkz): x-FFT, the aft.py:203-206 /
// sekspace.py:198-206 multiplier, inverse x-FFT in one pass; a second
// all-to-all and the inverse 2-D C2R return the x-slab.  Forward transforms
// are unnormalised; the multiplier carries 1/M^3 as in the replicated path.

__global__ void swap01_kernel(const cplx *__restrict__ src, int a, int b, int64_t c, cplx *__restrict__ dst) {
    // dst (b, a, c) <- src (a, b, c)
    const int64_t total = (int64_t)a * b * c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i % c;
        const int64_t r = i / c;
        const int jb = (int)(r % b), ia = (int)(r / b);
        dst[((int64_t)jb * a + ia) * c + k] = src[i];
    }
}

__global__ void scale_slab_kernel(cplx *__restrict__ F, int M, int nky, int ky0, const double *__restrict__ k,
                                  const double *__restrict__ w, double xi, double norm) {
    const int nh = M / 2 + 1;
    const int64_t total = (int64_t)M * nky * nh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int iz = (int)(i % nh);
        const int64_t r = i / nh;
        const int iy = ky0 + (int)(r % nky), ix = (int)(r / nky);
        const double k2 = k[ix] * k[ix] + k[iy] * k[iy] + k[iz] * k[iz];
        const double W = w[ix] * w[iy] * w[iz];
        const double fac = k2 > 0.0 ? 4.0 * M_PI * mollify(k2, xi) * (1.0 / k2) / (W * W) * norm : 0.0;
        const cplx v = F[i];
        F[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// D = 0 (truncated-kernel path): F *= ghat * 4 pi af[kx] af[ky] ah[kz] / n^3 on
// this rank's ky-chunk of the (kx, ky, kz) spectrum (layout (n, nky, nh))
__global__ void scale_d0k_slab_kernel(cplx *__restrict__ F, int n, int nky, int ky0, const double *__restrict__ ghat,
                                      const double *__restrict__ af, const double *__restrict__ ah, double norm) {
    const int nh = n / 2 + 1;
    const int64_t total = (int64_t)n * nky * nh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int iz = (int)(i % nh);
        const int64_t r = i / nh;
        const int iy = ky0 + (int)(r % nky), ix = (int)(r / nky);
        const double fac = ghat[((int64_t)ix * n + iy) * nh + iz] * (4.0 * M_PI * af[ix]) * af[iy] * ah[iz] * norm;
        const cplx v = F[i];
        F[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// Slab-decomposed k-space stage: D = 3 on the M^3 grid; D = 0 (the
// truncated-kernel path, sekspace.py:301-337) on the nconv^3 zero-padded
// grid, whose x-planes >= Mt are zero.  n = M or nconv; rank r owns x-planes
// [r n / world, (r + 1) n / world) and, after the transpose, ky-chunk r.
static int slab_n(se_plan *pl) {
    if (pl->D == 3) return pl->g.M;
    if (pl->D == 0) return d0_geometry(pl->g.L, pl->g.M, pl->g.P, pl->p.s0, pl->p.rc, true).nconv;
    fail(SE_EINVAL, "the slab-decomposed k-space stage covers D = 3 and the D = 0 kernel path");
    return 0;
}

void slab_geometry(se_plan *pl, int world, int64_t *nx, int64_t *nky, int64_t *nkz) {
    const int n = slab_n(pl);
    if (world < 1 || n % world)
        fail(SE_EINVAL, "slab decomposition needs the transform size (M, or nconv for D = 0) divisible by the ranks");
    *nx = n / world;
    *nky = n / world;
    *nkz = n / 2 + 1;
}

static void slab_ffts(se_plan *pl, int world) {
    if (pl->slab_world == world) return;
    for (cufftHandle *h : {&pl->slab_f2, &pl->slab_i2, &pl->slab_x}) {
        if (*h) cufftDestroy(*h);
        *h = 0;
    }
    const int n = slab_n(pl), nx = n / world, nky = n / world, nh = n / 2 + 1;
    int n2[2] = {n, n}, rin[2] = {n, n}, cout[2] = {n, nh};
    SE_CUFFT(cufftPlanMany(&pl->slab_f2, 2, n2, rin, 1, n * n, cout, 1, n * nh, CUFFT_D2Z, nx));
    SE_CUFFT(cufftPlanMany(&pl->slab_i2, 2, n2, cout, 1, n * nh, rin, 1, n * n, CUFFT_Z2D, nx));
    int n1[1] = {n}, e1[1] = {n};
    SE_CUFFT(cufftPlanMany(&pl->slab_x, 1, n1, e1, nky * nh, 1, e1, nky * nh, 1, CUFFT_Z2Z, nky * nh));
    pl->slab_world = world;
}

// slab: (nx, M, M) real for D = 3; for D = 0 the (nx, Mt, Mt) planes of the
// spread grid (zero for planes >= Mt), zero-padded to (nx, n, n) here
void slab_forward(se_plan *pl, int world, const double *slab, double *send) {
    int64_t nx, nky, nkz;
    slab_geometry(pl, world, &nx, &nky, &nkz);
    slab_ffts(pl, world);
    set_streams(pl, {pl->slab_f2});
    const int n = slab_n(pl);
    pl->spec.ensure(sizeof(cplx) * (size_t)nx * n * nkz);
    const double *src = slab;
    if (pl->D == 0) {
        const int Mt = pl->g.Mt;
        pl->grid_tmp.ensure(sizeof(double) * (size_t)nx * n * n);
        LAUNCH(pad_real_kernel, nx * n * n, slab, (int)nx, Mt, Mt, pl->grid_tmp.as<double>(), (int)nx, n, n);
        src = pl->grid_tmp.as<double>();
    }
    SE_CUFFT(cufftExecD2Z(pl->slab_f2, const_cast<double *>(src), pl->spec.as<cplx>()));
    // (nx, world, nky * nkz) -> (world, nx, nky * nkz)
    LAUNCH(swap01_kernel, nx * n * nkz, pl->spec.as<cplx>(), (int)nx, world, nky * nkz, reinterpret_cast<cplx *>(send));
}

void slab_xpass(se_plan *pl, int world, int rank, double *recv) {
    int64_t nx, nky, nkz;
    slab_geometry(pl, world, &nx, &nky, &nkz);
    if (rank < 0 || rank >= world) fail(SE_EINVAL, "rank out of range");
    ensure_tables(pl);
    if (pl->D == 0) d0_kernel_prepare(pl, nullptr);
    slab_ffts(pl, world);
    set_streams(pl, {pl->slab_x});
    const int n = slab_n(pl);
    cplx *F = reinterpret_cast<cplx *>(recv);
    SE_CUFFT(cufftExecZ2Z(pl->slab_x, F, F, CUFFT_FORWARD));
    if (pl->D == 3)
        LAUNCH(scale_slab_kernel, (int64_t)n * nky * nkz, F, n, (int)nky, (int)(rank * nky), pl->tM.k.as<double>(),
               pl->tM.what.as<double>(), pl->p.xi, 1.0 / ((double)n * n * n));
    else
        LAUNCH(scale_d0k_slab_kernel, (int64_t)n * nky * nkz, F, n, (int)nky, (int)(rank * nky), pl->ghat.as<double>(),
               pl->tNc.what.as<double>(), pl->tNh.what.as<double>(), 1.0 / ((double)n * n * n));
    SE_CUFFT(cufftExecZ2Z(pl->slab_x, F, F, CUFFT_INVERSE));
}

// back (world, nx, nky, nkz) -> slab: (nx, M, M) for D = 3, the (nx, Mt, Mt)
// restriction of the padded planes for D = 0
void slab_inverse(se_plan *pl, int world, const double *back, double *slab) {
    int64_t nx, nky, nkz;
    slab_geometry(pl, world, &nx, &nky, &nkz);
    slab_ffts(pl, world);
    set_streams(pl, {pl->slab_i2});
    const int n = slab_n(pl);
    pl->spec.ensure(sizeof(cplx) * (size_t)nx * n * nkz);
    // (world, nx, nky * nkz) -> (nx, world, nky * nkz) = (nx, n, nkz)
    LAUNCH(swap01_kernel, nx * n * nkz, reinterpret_cast<const cplx *>(back), world, (int)nx, nky * nkz,
           pl->spec.as<cplx>());
    if (pl->D == 3) {
        SE_CUFFT(cufftExecZ2D(pl->slab_i2, pl->spec.as<cplx>(), slab));
        return;
    }
    const int Mt = pl->g.Mt;
    pl->grid_tmp.ensure(sizeof(double) * (size_t)nx * n * n);
    SE_CUFFT(cufftExecZ2D(pl->slab_i2, pl->spec.as<cplx>(), pl->grid_tmp.as<double>()));
    LAUNCH(restrict_real_kernel, nx * Mt * Mt, pl->grid_tmp.as<double>(), n, n, slab, (int)nx, Mt, Mt, 1.0);
}

// ------------------------------------ row-distributed adaptive FFT (D = 1, 2)
// The AFT of D in {1, 2} (aft.py:168-265, sekspace.py:217-254) over `world`
// ranks: rank r holds the z-chunk z in [nz0, nz0 + nz) of the
// grid (every x, y): the periodic R2C (2-D over (x, y) for D = 2, 1-D over x
// for D = 1) is local to a z-plane; its output rows (periodic modes, the
// halved axis last) are grouped by row chunk, so an all-to-all hands rank d
// every z of its rows [row0, row0 + nrows); there the free-axis blocks (zero
// mode padded to g0, I rows to gs, J rows at Mt) are transformed, scaled and
// inverted exactly as in the single-GPU stage, and the reverse all-to-all and
// the inverse periodic C2R return the filtered z-chunk.
//   rows: D = 2: (kx, ky) with ky < M/2 + 1, chunks of (M / world) kx values;
//         D = 1: kx < M/2 + 1, chunks of ceil((M/2 + 1) / world);
//   a row carries per_y x Mt values (per_y = 1 for D = 2, Mt for D = 1).
struct ZGeom {
    int nz0, nz, row0, nrows, rows_total, per_y;
};

static ZGeom zslab_geom(const se_plan *pl, int world, int rank) {
    const int D = pl->D, M = pl->g.M, Mt = pl->g.Mt, half = M / 2 + 1;
    if (D != 1 && D != 2) fail(SE_EINVAL, "the row-distributed AFT covers D = 1 and D = 2");
    if (world < 1 || rank < 0 || rank >= world) fail(SE_EINVAL, "invalid (rank, world)");
    if (Mt < world) fail(SE_EINVAL, "more ranks than free-axis planes");
    ZGeom z{};
    z.nz0 = (int)((int64_t)Mt * rank / world);
    z.nz = (int)((int64_t)Mt * (rank + 1) / world) - z.nz0;
    if (D == 2) {
        if (M % world) fail(SE_EINVAL, "the row-distributed AFT of D = 2 needs M divisible by the ranks");
        z.rows_total = M * half;
        z.nrows = (M / world) * half;
        z.row0 = rank * z.nrows;
        z.per_y = 1;
    } else {
        const int c = (half + world - 1) / world;
        z.rows_total = half;
        z.row0 = std::min(rank * c, half);
        z.nrows = std::min(half, z.row0 + c) - z.row0;
        z.per_y = Mt;
    }
    return z;
}

static void zslab_plans(se_plan *pl, int world, int rank) {
    if (pl->zs_world == world && pl->zs_rank == rank) return;
    for (cufftHandle *h : {&pl->zs_fwd, &pl->zs_inv, &pl->zs_rowJ, &pl->zs_rowI, &pl->zs_row0}) {
        if (*h) cufftDestroy(*h);
        *h = 0;
    }
    ensure_tables(pl);
    const ZGeom z = zslab_geom(pl, world, rank);
    const se_grid_t &g = pl->g;
    const int D = pl->D, M = g.M, Mt = g.Mt, half = M / 2 + 1;
    if (D == 2) {
        int n[2] = {M, M}, rin[2] = {M, M}, cout[2] = {M, half};
        SE_CUFFT(cufftPlanMany(&pl->zs_fwd, 2, n, rin, z.nz, 1, cout, z.nz, 1, CUFFT_D2Z, z.nz));
        SE_CUFFT(cufftPlanMany(&pl->zs_inv, 2, n, cout, z.nz, 1, rin, z.nz, 1, CUFFT_Z2D, z.nz));
    } else {
        int n[1] = {M}, rin[1] = {M}, cout[1] = {half};
        const int lines = Mt * z.nz;
        SE_CUFFT(cufftPlanMany(&pl->zs_fwd, 1, n, rin, lines, 1, cout, lines, 1, CUFFT_D2Z, lines));
        SE_CUFFT(cufftPlanMany(&pl->zs_inv, 1, n, cout, lines, 1, rin, lines, 1, CUFFT_Z2D, lines));
    }
    // this chunk's I rows (local indices) and the zero row (global row 0)
    std::vector<int> m = signed_modes(M), rows;
    for (int lr = 0; lr < z.nrows; ++lr) {
        const int row = z.row0 + lr;
        int mu;
        if (D == 2) {
            const int ix = row / half, iy = row - ix * half;
            mu = std::max(std::abs(m[ix]), std::abs(m[iy]));
        } else {
            mu = std::abs(m[row]);
        }
        if (mu >= 1 && mu <= pl->p.nI) rows.push_back(lr);
    }
    pl->zs_nI = (int)rows.size();
    pl->zs_rowsI.ensure(sizeof(int) * (rows.size() + 1));
    if (!rows.empty())
        SE_CUDA(cudaMemcpy(pl->zs_rowsI.ptr, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    if (D == 2) {
        int nJ[1] = {Mt}, nI1[1] = {g.gs}, n0[1] = {g.g0};
        if (z.nrows > 0)
            SE_CUFFT(cufftPlanMany(&pl->zs_rowJ, 1, nJ, nullptr, 1, Mt, nullptr, 1, Mt, CUFFT_Z2Z, z.nrows));
        if (pl->zs_nI > 0)
            SE_CUFFT(cufftPlanMany(&pl->zs_rowI, 1, nI1, nullptr, 1, g.gs, nullptr, 1, g.gs, CUFFT_Z2Z, pl->zs_nI));
        SE_CUFFT(cufftPlanMany(&pl->zs_row0, 1, n0, nullptr, 1, g.g0, nullptr, 1, g.g0, CUFFT_Z2Z, 1));
        pl->zs_Z.ensure(sizeof(cplx) * (size_t)g.g0);
        pl->zs_B.ensure(sizeof(cplx) * (size_t)(pl->zs_nI ? pl->zs_nI : 1) * g.gs);
    } else {
        int nJ[2] = {Mt, Mt}, nI2[2] = {g.gs, g.gs}, n0[2] = {g.g0, g.g0};
        if (z.nrows > 0)
            SE_CUFFT(cufftPlanMany(&pl->zs_rowJ, 2, nJ, nullptr, 1, Mt * Mt, nullptr, 1, Mt * Mt, CUFFT_Z2Z, z.nrows));
        if (pl->zs_nI > 0)
            SE_CUFFT(cufftPlanMany(&pl->zs_rowI, 2, nI2, nullptr, 1, g.gs * g.gs, nullptr, 1, g.gs * g.gs, CUFFT_Z2Z,
                                   pl->zs_nI));
        SE_CUFFT(cufftPlanMany(&pl->zs_row0, 2, n0, nullptr, 1, g.g0 * g.g0, nullptr, 1, g.g0 * g.g0, CUFFT_Z2Z, 1));
        pl->zs_Z.ensure(sizeof(cplx) * (size_t)g.g0 * g.g0);
        pl->zs_B.ensure(sizeof(cplx) * (size_t)(pl->zs_nI ? pl->zs_nI : 1) * g.gs * g.gs);
    }
    pl->zs_Hk.ensure(sizeof(cplx) * ((size_t)z.nrows * z.per_y * Mt + 1));
    pl->zs_world = world;
    pl->zs_rank = rank;
}

// recv [source s][my rows][per_y][nz_s] <-> Hk [my rows][per_y][Mt] (z of
// source s at [nz0_s, nz0_s + nz_s), nz0_s = Mt s / world)
template <bool TO_ROWS>
__global__ void zslab_reorder_kernel(cplx *__restrict__ recv, cplx *__restrict__ Hk, int64_t nrows_py, int Mt,
                                     int world) {
    const int64_t total = nrows_py * Mt;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(i % Mt);
        const int64_t rp = i / Mt;
        int s = 0;
        while (s + 1 < world && (int)((int64_t)Mt * (s + 1) / world) <= z) ++s;
        const int nz0 = (int)((int64_t)Mt * s / world), nz = (int)((int64_t)Mt * (s + 1) / world) - nz0;
        const int64_t j = nrows_py * nz0 + rp * nz + (z - nz0);
        if (TO_ROWS)
            Hk[i] = recv[j];
        else
            recv[j] = Hk[i];
    }
}

void zslab_geometry(se_plan *pl, int world, int rank, int64_t *out) {
    const ZGeom z = zslab_geom(pl, world, rank);
    out[0] = z.nz0;
    out[1] = z.nz;
    out[2] = z.row0;
    out[3] = z.nrows;
    out[4] = z.rows_total;
    out[5] = z.per_y;
}

// zslab (M, M or Mt, nz) real -> spec (rows_total, per_y, nz) complex
void zslab_forward(se_plan *pl, int world, int rank, const double *zslab, double *spec) {
    zslab_plans(pl, world, rank);
    set_streams(pl, {pl->zs_fwd});
    SE_CUFFT(cufftExecD2Z(pl->zs_fwd, const_cast<double *>(zslab), reinterpret_cast<cplx *>(spec)));
}

void zslab_inverse(se_plan *pl, int world, int rank, const double *spec, double *zslab) {
    zslab_plans(pl, world, rank);
    set_streams(pl, {pl->zs_inv});
    // cuFFT's C2R may overwrite its input: the caller's spectrum is scratch here
    SE_CUFFT(cufftExecZ2D(pl->zs_inv, reinterpret_cast<cplx *>(const_cast<double *>(spec)), zslab));
}

// in place on recv: this rank's rows, every z, through the free-axis blocks
void zslab_rows(se_plan *pl, int world, int rank, double *recv) {
    zslab_plans(pl, world, rank);
    const ZGeom z = zslab_geom(pl, world, rank);
    if (z.nrows <= 0) return;
    const se_grid_t &g = pl->g;
    const int D = pl->D, M = g.M, Mt = g.Mt, half = M / 2 + 1, nfree = 3 - D;
    set_streams(pl, {pl->zs_rowJ, pl->zs_rowI, pl->zs_row0});
    cplx *R = reinterpret_cast<cplx *>(recv), *Hk = pl->zs_Hk.as<cplx>(), *Z = pl->zs_Z.as<cplx>(),
         *B = pl->zs_B.as<cplx>();
    const int64_t nrp = (int64_t)z.nrows * z.per_y;
    LAUNCH(zslab_reorder_kernel<true>, nrp * Mt, R, Hk, nrp, Mt, world);
    const int *rows = pl->zs_rowsI.as<int>();
    const int nI = pl->zs_nI;
    const bool zero_here = z.row0 == 0;  // the k = 0 row lives in the first chunk
    MixArgs ma{D, M, pl->p.nI, half, pl->p.xi, g.R, pl->tM.k.as<double>(), pl->tM.what.as<double>()};
    ma.row0 = z.row0;
    ma.nrows = z.nrows;
    const double perN = D == 2 ? (double)M * M : (double)M;
    auto pw = [&](int n) { return nfree == 1 ? (double)n : (double)n * n; };
    if (zero_here) LAUNCH(pack_kernel, (int64_t)pw(g.g0), Hk, Mt, nfree, nullptr, 1, Z, g.g0);
    if (nI) LAUNCH(pack_kernel, (int64_t)pw(g.gs) * nI, Hk, Mt, nfree, rows, nI, B, g.gs);
    SE_CUFFT(cufftExecZ2Z(pl->zs_rowJ, Hk, Hk, CUFFT_FORWARD));
    if (nI) SE_CUFFT(cufftExecZ2Z(pl->zs_rowI, B, B, CUFFT_FORWARD));
    if (zero_here) SE_CUFFT(cufftExecZ2Z(pl->zs_row0, Z, Z, CUFFT_FORWARD));
    LAUNCH(scale_mixJ_kernel, (int64_t)z.nrows * (int64_t)pw(Mt), Hk, ma, Mt, pl->tMt.k.as<double>(),
           pl->tMt.what.as<double>(), 1.0 / (pw(Mt) * perN));
    if (nI)
        LAUNCH(scale_mixI_kernel, (int64_t)pw(g.gs) * nI, B, ma, rows, nI, g.gs, pl->tgs.k.as<double>(),
               pl->tgs.what.as<double>(), 1.0 / (pw(g.gs) * perN));
    if (zero_here)
        LAUNCH(scale_mix0_kernel, (int64_t)pw(g.g0), Z, ma, g.g0, pl->tg0.k.as<double>(), pl->tg0.what.as<double>(),
               1.0 / (pw(g.g0) * perN));
    SE_CUFFT(cufftExecZ2Z(pl->zs_rowJ, Hk, Hk, CUFFT_INVERSE));
    if (nI) SE_CUFFT(cufftExecZ2Z(pl->zs_rowI, B, B, CUFFT_INVERSE));
    if (zero_here) SE_CUFFT(cufftExecZ2Z(pl->zs_row0, Z, Z, CUFFT_INVERSE));
    if (nI) LAUNCH(unpack_kernel, (int64_t)pw(Mt) * nI, B, g.gs, nfree, rows, nI, Hk, Mt);
    if (zero_here) LAUNCH(unpack_kernel, (int64_t)pw(Mt), Z, g.g0, nfree, nullptr, 1, Hk, Mt);
    LAUNCH(zslab_reorder_kernel<false>, nrp * Mt, R, Hk, nrp, Mt, world);
}

// ------------------------------------------------------ field (D = 3, ik)
// E_F = -grad phi_F by spectral differentiation of the filtered grid: the
// gather is a convolution with the window, so grad commutes with it and
// E_F,a = gather(IFFT(-i k_a Phi)), Phi the scaled spectrum (three inverse
// transforms, three gathers; no window derivative -- the ES window's is
// singular at the support edge).  The Nyquist plane of the differentiated
// axis is zeroed (real output).
__global__ void grad_d3_kernel(const cplx *__restrict__ F, cplx *__restrict__ G, int M, const double *__restrict__ k,
                               int axis) {
    const int nh = M / 2 + 1;
    const int64_t total = (int64_t)M * M * nh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int iz = (int)(i % nh);
        const int64_t r = i / nh;
        const int iy = (int)(r % M), ix = (int)(r / M);
        const int id = axis == 0 ? ix : (axis == 1 ? iy : iz);
        const double kk = id == M / 2 ? 0.0 : k[id];
        const cplx v = F[i];
        G[i] = make_double2(kk * v.y, -kk * v.x);  // -i k (re + i im)
    }
}

void kspace_field_run(se_plan *pl, double *grid, double *g3) {
    if (pl->D != 3) fail(SE_EINVAL, "the electric field (forces) covers D = 3");
    ensure_tables(pl);
    make_ffts(pl);
    set_streams(pl, {pl->fft_fwd, pl->fft_inv});
    const int M = pl->g.M;
    const size_t G = (size_t)M * M * M, S = (size_t)M * M * (M / 2 + 1);
    pl->spec2.ensure(sizeof(cplx) * S);
    SE_CUFFT(cufftExecD2Z(pl->fft_fwd, grid, pl->spec.as<cplx>()));
    LAUNCH(scale_d3_kernel, (int64_t)S, pl->spec.as<cplx>(), M, pl->tM.k.as<double>(), pl->tM.what.as<double>(),
           pl->p.xi, 1.0 / ((double)M * M * M));
    for (int a = 0; a < 3; ++a) {
        LAUNCH(grad_d3_kernel, (int64_t)S, pl->spec.as<cplx>(), pl->spec2.as<cplx>(), M, pl->tM.k.as<double>(), a);
        SE_CUFFT(cufftExecZ2D(pl->fft_inv, pl->spec2.as<cplx>(), g3 + a * G));
    }
}

}  // namespace se
