// Stage-level entry points that the reference exposes module by module:
//  * the FFT engine plugin (aft.py:24-53: fftn / ifftn / rfftn / irfftn with
//    numpy semantics) on cuFFT, for a contiguous block of axes of a
//    C-ordered array (outer dims looped, inner dims batched);
//  * sekspace.scale (sekspace.py:192-254) on a SpectralField in the
//    reference's block layout (D=3 full, D=0 zero block, D in {1,2} zero /
//    I rows / J rows with explicit periodic-mode row indices).
// The hot pipeline (se_kspace_apply) does not use these: it keeps R2C half
// spectra on the device.  These serve the reference's stage API and tests.
#include <cufft.h>

#include <vector>

#include "se_common.h"

namespace se {

typedef double2 cplx;

namespace {

struct FftShape {
    long long outer = 1, inner = 1;
    std::vector<int> n;  // transformed dims
};

FftShape split_axes(int ndim, const int64_t *shape, int ax0, int ax1) {
    if (ndim < 1 || ax0 < 0 || ax1 >= ndim || ax0 > ax1) fail(SE_EINVAL, "invalid FFT axes");
    FftShape f;
    for (int i = 0; i < ax0; ++i) f.outer *= shape[i];
    for (int i = ax1 + 1; i < ndim; ++i) f.inner *= shape[i];
    for (int i = ax0; i <= ax1; ++i) {
        if (shape[i] < 1 || shape[i] > (1 << 30)) fail(SE_EINVAL, "invalid FFT length");
        f.n.push_back((int)shape[i]);
    }
    return f;
}

long long prod(const std::vector<int> &v) {
    long long p = 1;
    for (int x : v) p *= x;
    return p;
}

__global__ void scale_inplace_kernel(cplx *a, long long n, double s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        cplx v = a[i];
        a[i] = make_double2(v.x * s, v.y * s);
    }
}

__global__ void scale_real_kernel(double *a, long long n, double s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a[i] *= s;
}

unsigned blocks_for(long long n) {
    long long b = (n + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

void check_device(int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        fail(SE_EDEVICE, "no CUDA device available (the SE B200 library has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) fail(SE_EINVAL, "device ordinal out of range");
    SE_CUDA(cudaSetDevice(device));
}

struct Tmp {
    void *p = nullptr;
    ~Tmp() {
        if (p) cudaFree(p);
    }
};

}  // namespace

// ---------------------------------------------------------- block multiplier
struct ScaleArgs {
    int D, M, Mt, g0, gs;
    double xi, R;
};

__device__ __forceinline__ double mollifier(double k2, double xi) { return exp(-k2 / (4.0 * xi * xi)); }
__device__ double greens_zero_dev2(int D, double R, double kappa);

// D=3 full (M^3) or D=0 zero block (g0^3): sekspace.py:198-215
__global__ void stage_scale_cube_kernel(cplx *F, int n, const double *k, const double *w, ScaleArgs a) {
    long long total = (long long)n * n * n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        int iz = (int)(i % n);
        long long r = i / n;
        int iy = (int)(r % n), ix = (int)(r / n);
        double k2 = k[ix] * k[ix] + k[iy] * k[iy] + k[iz] * k[iz];
        double W = w[ix] * w[iy] * w[iz];
        double g;
        if (a.D == 3)
            g = k2 > 0.0 ? 1.0 / k2 : 0.0;
        else
            g = greens_zero_dev2(0, a.R, sqrt(k2));
        double fac = 4.0 * M_PI * mollifier(k2, a.xi) * g / (W * W);
        cplx v = F[i];
        F[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// zero block of D in {1,2}: sekspace.py:221-232
__global__ void stage_scale_zero_kernel(cplx *Z, ScaleArgs a, const double *kf, const double *wf, double wp0) {
    const int nfree = 3 - a.D, g = a.g0;
    long long total = nfree == 1 ? g : (long long)g * g;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        double kap2, wfree;
        if (nfree == 1) {
            kap2 = kf[i] * kf[i];
            wfree = wf[i];
        } else {
            int y = (int)(i / g), z = (int)(i % g);
            kap2 = kf[y] * kf[y] + kf[z] * kf[z];
            wfree = wf[y] * wf[z];
        }
        double W = (a.D == 2 ? wp0 * wp0 : wp0) * wfree;
        double fac = 4.0 * M_PI * mollifier(kap2, a.xi) * greens_zero_dev2(a.D, a.R, sqrt(kap2)) / (W * W);
        cplx v = Z[i];
        Z[i] = make_double2(v.x * fac, v.y * fac);
    }
}

// I or J rows (explicit periodic indices, D ints per row): sekspace.py:234-254
__global__ void stage_scale_rows_kernel(cplx *B, int nrows, const int *idx, int glen, ScaleArgs a, const double *kp,
                                        const double *wp, const double *kf, const double *wf) {
    const int nfree = 3 - a.D;
    long long per = nfree == 1 ? glen : (long long)glen * glen;
    long long total = per * nrows;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        int r = (int)(i / per);
        long long e = i - (long long)r * per;
        double kr2, wr;
        if (a.D == 2) {
            int ix = idx[2 * r], iy = idx[2 * r + 1];
            kr2 = kp[ix] * kp[ix] + kp[iy] * kp[iy];
            wr = wp[ix] * wp[iy];
        } else {
            int ix = idx[r];
            kr2 = kp[ix] * kp[ix];
            wr = wp[ix];
        }
        double k2, W;
        if (nfree == 1) {
            k2 = kr2 + kf[e] * kf[e];
            W = wr * wf[e];
        } else {
            int y = (int)(e / glen), z = (int)(e % glen);
            k2 = kr2 + kf[y] * kf[y] + kf[z] * kf[z];
            W = wr * (wf[y] * wf[z]);
        }
        double fac = 4.0 * M_PI * mollifier(k2, a.xi) / (k2 * (W * W));
        cplx v = B[i];
        B[i] = make_double2(v.x * fac, v.y * fac);
    }
}

__device__ double greens_zero_dev2(int D, double R, double kappa) {
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

}  // namespace se

using namespace se;

#define SE_API_BEGIN try {
#define SE_API_END                    \
    return SE_OK;                     \
    }                                 \
    catch (const se::Error &e) {      \
        se::set_last_error(e.what()); \
        return e.code;                \
    }                                 \
    catch (const std::exception &e) { \
        se::set_last_error(e.what()); \
        return SE_EDEVICE;            \
    }

extern "C" {

int se_fft_c2c_host(int device, int ndim, const int64_t *shape, int ax0, int ax1, int inverse, const double *in,
                    double *out) {
    SE_API_BEGIN
    check_device(device);
    FftShape f = split_axes(ndim, shape, ax0, ax1);
    const long long per = prod(f.n) * f.inner, total = per * f.outer;
    Tmp buf;
    SE_CUDA(cudaMalloc(&buf.p, sizeof(cplx) * (total ? total : 1)));
    cplx *d = (cplx *)buf.p;
    SE_CUDA(cudaMemcpy(d, in, sizeof(cplx) * total, cudaMemcpyHostToDevice));
    cufftHandle h = 0;
    std::vector<int> n = f.n;
    SE_CUFFT(cufftPlanMany(&h, (int)n.size(), n.data(), n.data(), (int)f.inner, 1, n.data(), (int)f.inner, 1, CUFFT_Z2Z,
                           (int)f.inner));
    for (long long o = 0; o < f.outer; ++o) {
        cufftResult r = cufftExecZ2Z(h, d + o * per, d + o * per, inverse ? CUFFT_INVERSE : CUFFT_FORWARD);
        if (r != CUFFT_SUCCESS) {
            cufftDestroy(h);
            fail(SE_EDEVICE, "cuFFT Z2Z failed");
        }
    }
    cufftDestroy(h);
    if (inverse && total) scale_inplace_kernel<<<blocks_for(total), 256>>>(d, total, 1.0 / (double)prod(f.n));
    SE_CUDA(cudaMemcpy(out, d, sizeof(cplx) * total, cudaMemcpyDeviceToHost));
    SE_API_END
}

int se_fft_r2c_host(int device, int ndim, const int64_t *shape, int ax0, int ax1, const double *in, double *out) {
    SE_API_BEGIN
    check_device(device);
    if (ax1 != ndim - 1) fail(SE_EINVAL, "r2c transforms need the last axis among the transformed axes");
    FftShape f = split_axes(ndim, shape, ax0, ax1);
    std::vector<int> nh = f.n;
    nh.back() = f.n.back() / 2 + 1;
    const long long rin = prod(f.n), cout = prod(nh);
    Tmp bi, bo;
    SE_CUDA(cudaMalloc(&bi.p, sizeof(double) * (rin * f.outer ? rin * f.outer : 1)));
    SE_CUDA(cudaMalloc(&bo.p, sizeof(cplx) * (cout * f.outer ? cout * f.outer : 1)));
    SE_CUDA(cudaMemcpy(bi.p, in, sizeof(double) * rin * f.outer, cudaMemcpyHostToDevice));
    cufftHandle h = 0;
    std::vector<int> n = f.n;
    SE_CUFFT(cufftPlanMany(&h, (int)n.size(), n.data(), nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, (int)f.outer));
    cufftResult r = cufftExecD2Z(h, (double *)bi.p, (cplx *)bo.p);
    cufftDestroy(h);
    if (r != CUFFT_SUCCESS) fail(SE_EDEVICE, "cuFFT D2Z failed");
    SE_CUDA(cudaMemcpy(out, bo.p, sizeof(cplx) * cout * f.outer, cudaMemcpyDeviceToHost));
    SE_API_END
}

int se_fft_c2r_host(int device, int ndim, const int64_t *out_shape, int ax0, int ax1, const double *in, double *out) {
    SE_API_BEGIN
    check_device(device);
    if (ax1 != ndim - 1) fail(SE_EINVAL, "c2r transforms need the last axis among the transformed axes");
    FftShape f = split_axes(ndim, out_shape, ax0, ax1);
    std::vector<int> nh = f.n;
    nh.back() = f.n.back() / 2 + 1;
    const long long rout = prod(f.n), cin = prod(nh);
    Tmp bi, bo;
    SE_CUDA(cudaMalloc(&bi.p, sizeof(cplx) * (cin * f.outer ? cin * f.outer : 1)));
    SE_CUDA(cudaMalloc(&bo.p, sizeof(double) * (rout * f.outer ? rout * f.outer : 1)));
    SE_CUDA(cudaMemcpy(bi.p, in, sizeof(cplx) * cin * f.outer, cudaMemcpyHostToDevice));
    cufftHandle h = 0;
    std::vector<int> n = f.n;
    SE_CUFFT(cufftPlanMany(&h, (int)n.size(), n.data(), nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, (int)f.outer));
    cufftResult r = cufftExecZ2D(h, (cplx *)bi.p, (double *)bo.p);
    cufftDestroy(h);
    if (r != CUFFT_SUCCESS) fail(SE_EDEVICE, "cuFFT Z2D failed");
    if (rout * f.outer) scale_real_kernel<<<blocks_for(rout * f.outer), 256>>>((double *)bo.p, rout * f.outer, 1.0 / (double)rout);
    SE_CUDA(cudaMemcpy(out, bo.p, sizeof(double) * rout * f.outer, cudaMemcpyDeviceToHost));
    SE_API_END
}

// sekspace.scale on host blocks.  tables: kp/wp (M periodic modes),
// k0/w0 (g0 modes), ks/ws (gs modes), kt/wt (Mt modes) -- wavenumbers and
// window transforms; for D=3 only kp/wp (M), for D=0 only k0/w0 (g0).
int se_scale_blocks_host(int device, int D, int M, int Mt, int g0, int gs, double xi, double R, const double *kp,
                         const double *wp, const double *k0, const double *w0, const double *ks, const double *ws,
                         const double *kt, const double *wt, double *cube_or_zero, double *Iblk, const int *I_idx,
                         int64_t nI, double *Jblk, const int *J_idx, int64_t nJ) {
    SE_API_BEGIN
    check_device(device);
    if (D < 0 || D > 3) fail(SE_EINVAL, "D must be in {0,1,2,3}");
    ScaleArgs a{D, M, Mt, g0, gs, xi, R};
    std::vector<void *> frees;
    auto up = [&](const void *h, size_t bytes) -> void * {
        void *d = nullptr;
        SE_CUDA(cudaMalloc(&d, bytes ? bytes : 8));
        frees.push_back(d);
        if (bytes) SE_CUDA(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
        return d;
    };
    struct Guard {
        std::vector<void *> &v;
        ~Guard() {
            for (void *p : v) cudaFree(p);
        }
    } guard{frees};
    if (D == 3 || D == 0) {
        const int n = D == 3 ? M : g0;
        const double *kk = D == 3 ? kp : k0, *ww = D == 3 ? wp : w0;
        long long tot = (long long)n * n * n;
        cplx *dF = (cplx *)up(cube_or_zero, sizeof(cplx) * tot);
        stage_scale_cube_kernel<<<blocks_for(tot), 256>>>(dF, n, (double *)up(kk, 8 * n), (double *)up(ww, 8 * n), a);
        SE_LAUNCH_CHECK();
        SE_CUDA(cudaMemcpy(cube_or_zero, dF, sizeof(cplx) * tot, cudaMemcpyDeviceToHost));
        return SE_OK;
    }
    const int nfree = 3 - D;
    auto per = [&](int g) { return nfree == 1 ? (long long)g : (long long)g * g; };
    double *dkp = (double *)up(kp, 8 * M), *dwp = (double *)up(wp, 8 * M);
    // zero block
    {
        long long tot = per(g0);
        cplx *dZ = (cplx *)up(cube_or_zero, sizeof(cplx) * tot);
        stage_scale_zero_kernel<<<blocks_for(tot), 256>>>(dZ, a, (double *)up(k0, 8 * g0), (double *)up(w0, 8 * g0), wp[0]);
        SE_LAUNCH_CHECK();
        SE_CUDA(cudaMemcpy(cube_or_zero, dZ, sizeof(cplx) * tot, cudaMemcpyDeviceToHost));
    }
    auto rows = [&](double *blk, const int *idx, int64_t nr, int glen, const double *kf, const double *wf) {
        if (nr <= 0) return;
        long long tot = per(glen) * nr;
        cplx *dB = (cplx *)up(blk, sizeof(cplx) * tot);
        int *dI = (int *)up(idx, sizeof(int) * D * nr);
        stage_scale_rows_kernel<<<blocks_for(tot), 256>>>(dB, (int)nr, dI, glen, a, dkp, dwp, (double *)up(kf, 8 * glen),
                                                          (double *)up(wf, 8 * glen));
        SE_LAUNCH_CHECK();
        SE_CUDA(cudaMemcpy(blk, dB, sizeof(cplx) * tot, cudaMemcpyDeviceToHost));
    };
    rows(Iblk, I_idx, nI, gs, ks, ws);
    rows(Jblk, J_idx, nJ, Mt, kt, wt);
    SE_API_END
}

}  // extern "C"
