// Demag tensor setup on the device (once per context), fp64 throughout.
//
// K0a  k_tensor_octant: K = -N over the non-negative displacement octant
//      [0,nx) x [0,ny) x [0,nz) (the reference evaluates the same octant and
//      mirrors it, demag.hpp:66-88).  Near field: the Newell-Williams-Dunlop
//      f/g 27-point stencil (newell.cpp:31-209) in fp64 with Neumaier sums.
//      Far field: the exact cell-pair average written as a tent-weighted
//      integral of the point-dipole kernel, N(X) = (1/V) Int prod_i(d_i-|s_i|)
//      n(X+s) ds, evaluated by Gauss-Legendre quadrature (each tent split at
//      0).  This removes the eps*r^6 cancellation of the stencil that makes a
//      plain fp64 port 27% wrong at 300 cells.
// K0b  k_gemm64: the tensor spectrum is real with per-axis parity (all six
//      components are even or odd along each axis), so the padded 3-D DFT
//      of the mirrored lattice (demag.hpp:105-119) collapses to separable
//      cosine / sine transforms of the octant: three fp64 batched GEMMs
//      against C[u][d] = (d?2:1) cos(2 pi u d/P) or S[u][d] = 2 sin(2 pi u d/P).
#pragma once
#include "common.cuh"
#include "tensor_api.h"

namespace mfd {

// Gauss-Legendre nodes/weights on [-1,1] for n = 3..10 (mpmath, 22 digits).
__constant__ const double kGL[][2] = {
    // n = 3
    {-0.7745966692414833770359, 0.5555555555555555555556},
    {0.0, 0.8888888888888888888889},
    {0.7745966692414833770359, 0.5555555555555555555556},
    // n = 4
    {-0.8611363115940525752239, 0.3478548451374538573731},
    {-0.3399810435848562648027, 0.6521451548625461426269},
    {0.3399810435848562648027, 0.6521451548625461426269},
    {0.8611363115940525752239, 0.3478548451374538573731},
    // n = 5
    {-0.9061798459386639927976, 0.2369268850561890875143},
    {-0.5384693101056830910363, 0.4786286704993664680413},
    {0.0, 0.5688888888888888888889},
    {0.5384693101056830910363, 0.4786286704993664680413},
    {0.9061798459386639927976, 0.2369268850561890875143},
    // n = 6
    {-0.9324695142031520278123, 0.1713244923791703450403},
    {-0.6612093864662645136614, 0.3607615730481386075698},
    {-0.2386191860831969086305, 0.4679139345726910473899},
    {0.2386191860831969086305, 0.4679139345726910473899},
    {0.6612093864662645136614, 0.3607615730481386075698},
    {0.9324695142031520278123, 0.1713244923791703450403},
    // n = 7
    {-0.9491079123427585245262, 0.1294849661688696932706},
    {-0.7415311855993944398639, 0.2797053914892766679015},
    {-0.4058451513773971669066, 0.3818300505051189449504},
    {0.0, 0.4179591836734693877551},
    {0.4058451513773971669066, 0.3818300505051189449504},
    {0.7415311855993944398639, 0.2797053914892766679015},
    {0.9491079123427585245262, 0.1294849661688696932706},
    // n = 8
    {-0.9602898564975362316836, 0.1012285362903762591525},
    {-0.7966664774136267395916, 0.2223810344533744705444},
    {-0.5255324099163289858177, 0.313706645877887287338},
    {-0.1834346424956498049395, 0.3626837833783619829652},
    {0.1834346424956498049395, 0.3626837833783619829652},
    {0.5255324099163289858177, 0.313706645877887287338},
    {0.7966664774136267395916, 0.2223810344533744705444},
    {0.9602898564975362316836, 0.1012285362903762591525},
    // n = 9
    {-0.9681602395076260898356, 0.08127438836157441197189},
    {-0.8360311073266357942994, 0.1806481606948574040585},
    {-0.6133714327005903973087, 0.2606106964029354623187},
    {-0.3242534234038089290385, 0.3123470770400028400686},
    {0.0, 0.3302393550012597631645},
    {0.3242534234038089290385, 0.3123470770400028400686},
    {0.6133714327005903973087, 0.2606106964029354623187},
    {0.8360311073266357942994, 0.1806481606948574040585},
    {0.9681602395076260898356, 0.08127438836157441197189},
    // n = 10
    {-0.973906528517171720078, 0.06667134430868813759357},
    {-0.8650633666889845107321, 0.1494513491505805931458},
    {-0.6794095682990244062343, 0.2190863625159820439955},
    {-0.4333953941292471907993, 0.2692667193099963550912},
    {-0.1488743389816312108848, 0.2955242247147528701739},
    {0.1488743389816312108848, 0.2955242247147528701739},
    {0.4333953941292471907993, 0.2692667193099963550912},
    {0.6794095682990244062343, 0.2190863625159820439955},
    {0.8650633666889845107321, 0.1494513491505805931458},
    {0.973906528517171720078, 0.06667134430868813759357},

};
__host__ __device__ constexpr int gl_offset(int n) { return (n - 1) * n / 2 - 3; }

// ----------------------------------------------------------------- Newell fp64
__device__ double csum_d(const double* v, int n) {
    double s = v[0], c = 0.0;
    for (int i = 1; i < n; ++i) {
        const double t = s + v[i];
        c += fabs(s) >= fabs(v[i]) ? (s - t) + v[i] : (v[i] - t) + s;
        s = t;
    }
    return s + c;
}

__device__ double self_nx_d(double x, double y, double z) {
    if (x <= 0 || y <= 0 || z <= 0) return 0.0;
    if (x == y && y == z) return 1.0 / 3.0;
    const double x2 = x * x, y2 = y * y, z2 = z * z, R = sqrt(x2 + y2 + z2);
    const double dxy = (x - y) * (x + y), dxz = (x - z) * (x + z);
    double a[15];
    a[0] = -4.0 * (2.0 * x2 * x - y2 * y - z2 * z);
    a[1] = 4.0 * (x2 + dxy) * sqrt(x2 + y2);
    a[2] = 4.0 * (x2 + dxz) * sqrt(x2 + z2);
    a[3] = -4.0 * (y2 + z2) * sqrt(y2 + z2);
    a[4] = -4.0 * R * (dxy + dxz);
    a[5] = 24.0 * x * y * z * atan(y * z / (x * R));
    a[6] = 12.0 * (z + y) * x2 * log(x);
    a[7] = 12.0 * z * y2 * log((sqrt(y2 + z2) + z) / y);
    a[8] = -12.0 * z * x2 * log(sqrt(x2 + z2) + z);
    a[9] = 12.0 * z * dxy * log(R + z);
    a[10] = -6.0 * z * dxy * log(x2 + y2);
    a[11] = 12.0 * y * z2 * log((sqrt(y2 + z2) + y) / z);
    a[12] = -12.0 * y * x2 * log(sqrt(x2 + y2) + y);
    a[13] = 12.0 * y * dxz * log(R + y);
    a[14] = -6.0 * y * dxz * log(x2 + z2);
    return csum_d(a, 15) / (12.0 * M_PI * x * y * z);
}

__device__ double nf_d(double x, double y, double z) {
    x = fabs(x); y = fabs(y); z = fabs(z);
    const double x2 = x * x, y2 = y * y, z2 = z * z;
    double r = x2 + y2 + z2;
    if (r <= 0) return 0.0;
    r = sqrt(r);
    double p[8];
    int n = 0;
    if (z > 0) {
        p[n++] = 2.0 * (2.0 * x2 - y2 - z2) * r;
        if (x > 0 && y > 0) p[n++] = -12.0 * x * y * z * atan2(y * z, x * r);
        if (y > 0 && x2 + z2 > 0) {
            const double l = log(((y + r) * (y + r)) / (x2 + z2));
            p[n++] = 3.0 * y * z2 * l;
            p[n++] = -3.0 * y * x2 * l;
        }
        if (x2 + y2 > 0) {
            const double l = log(((z + r) * (z + r)) / (x2 + y2));
            p[n++] = 3.0 * z * y2 * l;
            p[n++] = -3.0 * z * x2 * l;
        }
    } else if (x == y) {
        p[n++] = -2.4598143973710680537922785 * x2 * x;   // 2 sqrt2 - 6 log(1+sqrt2)
    } else {
        p[n++] = 2.0 * (2.0 * x2 - y2) * r;
        if (y > 0 && x > 0) p[n++] = -6.0 * y * x2 * log((y + r) / x);
    }
    return csum_d(p, n) / 12.0;
}

__device__ double ng_d(double x, double y, double z) {
    double sg = 1.0;
    if (x < 0) sg = -sg;
    if (y < 0) sg = -sg;
    x = fabs(x); y = fabs(y); z = fabs(z);
    const double x2 = x * x, y2 = y * y, z2 = z * z;
    double r = x2 + y2 + z2;
    if (r <= 0) return 0.0;
    r = sqrt(r);
    double p[7];
    int n = 0;
    p[n++] = -2.0 * x * y * r;
    if (z > 0) {
        p[n++] = -z * z2 * atan2(x * y, z * r);
        p[n++] = -3.0 * z * y2 * atan2(x * z, y * r);
        p[n++] = -3.0 * z * x2 * atan2(y * z, x * r);
        if (x2 + y2 > 0) p[n++] = 6.0 * x * y * z * log((z + r) / sqrt(x2 + y2));
        if (y2 + z2 > 0) p[n++] = y * (3.0 * z2 - y2) * log((x + r) / sqrt(y2 + z2));
        if (x2 + z2 > 0) p[n++] = x * (3.0 * z2 - x2) * log((y + r) / sqrt(x2 + z2));
    } else {
        if (y > 0) p[n++] = -y * y2 * log((x + r) / y);
        if (x > 0) p[n++] = -x * x2 * log((y + r) / x);
    }
    return sg * csum_d(p, n) / 6.0;
}

template <bool G>
__device__ double stencil27_d(double x, double y, double z, double a, double b, double c) {
    // weights -1 (8 corners), +2 (12 edges), -4 (6 faces), +8 (centre)
    double v[27];
    int t = 0;
    for (int sx = -1; sx <= 1; ++sx)
        for (int sy = -1; sy <= 1; ++sy)
            for (int sz = -1; sz <= 1; ++sz) {
                const int nzero = (sx == 0) + (sy == 0) + (sz == 0);
                const double w = nzero == 0 ? -1.0 : nzero == 1 ? 2.0 : nzero == 2 ? -4.0 : 8.0;
                const double px = x + sx * a, py = y + sy * b, pz = z + sz * c;
                v[t++] = w * (G ? ng_d(px, py, pz) : nf_d(px, py, pz));
            }
    return csum_d(v, 27);
}

__device__ double newell_nxx(double X, double Y, double Z, double a, double b, double c) {
    if (X == 0 && Y == 0 && Z == 0) return self_nx_d(a, b, c);
    return stencil27_d<false>(X, Y, Z, a, b, c) / (4.0 * M_PI * a * b * c);
}
__device__ double newell_nxy(double X, double Y, double Z, double a, double b, double c) {
    return stencil27_d<true>(X, Y, Z, a, b, c) / (4.0 * M_PI * a * b * c);
}

// ---------------------------------------------------------- quadrature far field
// N(X) = (1/V) sum_nodes w_a w_b w_c n(X+s), n_xx = (r^2-3x^2)/(4 pi r^5), n_xy = -3xy/(4 pi r^5).
__device__ void gl_far(double X, double Y, double Z, double a, double b, double c, int n, double N6[6]) {
    double sx[20], wx[20], sy[20], wy[20], sz[20], wz[20];
    const int off = gl_offset(n);
    for (int q = 0; q < n; ++q) {
        const double xi = kGL[off + q][0], w = kGL[off + q][1];
        const double h = 0.5 * (1.0 + xi);          // node on [0,1]
        // [0, d] half: s = d*h, weight d/2*w, tent (d - s); mirrored half at -s
        sx[q] = a * h; wx[q] = 0.5 * a * w * (a - a * h);
        sy[q] = b * h; wy[q] = 0.5 * b * w * (b - b * h);
        sz[q] = c * h; wz[q] = 0.5 * c * w * (c - c * h);
        sx[n + q] = -sx[q]; wx[n + q] = wx[q];
        sy[n + q] = -sy[q]; wy[n + q] = wy[q];
        sz[n + q] = -sz[q]; wz[n + q] = wz[q];
    }
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 2 * n; ++i) {
        const double x = X + sx[i];
        double ai[6] = {0, 0, 0, 0, 0, 0};
        for (int j = 0; j < 2 * n; ++j) {
            const double y = Y + sy[j];
            double aj[6] = {0, 0, 0, 0, 0, 0};
            for (int k = 0; k < 2 * n; ++k) {
                const double z = Z + sz[k];
                const double r2 = x * x + y * y + z * z;
                const double ir = rsqrt(r2);
                const double ir2 = ir * ir;
                const double f = wz[k] * ir2 * ir2 * ir;   // w / r^5
                aj[0] += f * (r2 - 3.0 * x * x);
                aj[1] += f * (r2 - 3.0 * y * y);
                aj[2] += f * (r2 - 3.0 * z * z);
                aj[3] += f * x * y;
                aj[4] += f * x * z;
                aj[5] += f * y * z;
            }
            for (int q = 0; q < 6; ++q) ai[q] += wy[j] * aj[q];
        }
        for (int q = 0; q < 6; ++q) acc[q] += wx[i] * ai[q];
    }
    const double s = 1.0 / (4.0 * M_PI * a * b * c);
    N6[0] = acc[0] * s;
    N6[1] = acc[1] * s;
    N6[2] = acc[2] * s;
    N6[3] = -3.0 * acc[3] * s;
    N6[4] = -3.0 * acc[4] * s;
    N6[5] = -3.0 * acc[5] * s;
}

// Quadrature order for a displacement: the closest singularity of the
// dipole kernel lies D = max_i(|d_i|-1) d_i away; each half-tent interval
// of length d_max/2 then converges like rho^(-2n), rho = a + sqrt(a^2+1),
// a = 2D/d_max.  Returns 0 for "use exact Newell".
__device__ __host__ inline int far_order(int di, int dj, int dk, double a, double b, double c) {
    const double D = fmax(fmax((di - 1) * a, (dj - 1) * b), (dk - 1) * c);
    const double dm = fmax(fmax(a, b), c);
    const double q = 2.0 * D / dm;
    if (q < 6.0) return 0;
    const double rho = q + sqrt(q * q + 1.0);
    int n = (int)ceil(18.5 / log(rho));
    return n < 3 ? 3 : n > 10 ? 10 : n;
}

// K0a: one thread per octant entry; out layout [6][nz][ny][nx] (fp64).
// Planes [k0, k0 + nzc) of the octant; out = [6][nzc][ny][nx].
__global__ void k_tensor_octant(int nx, int ny, int k0, int nzc, double a, double b, double c,
                                double* __restrict__ out) {
    const long long n = (long long)nx * ny * nzc;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int i = (int)(e % nx), j = (int)((e / nx) % ny), k = k0 + (int)(e / ((long long)nx * ny));
    const double X = i * a, Y = j * b, Z = k * c;
    double K6[6];
    const int ord = far_order(i, j, k, a, b, c);
    if (ord == 0) {
        K6[0] = -newell_nxx(X, Y, Z, a, b, c);
        K6[1] = -newell_nxx(Y, Z, X, b, c, a);
        K6[2] = -newell_nxx(Z, X, Y, c, a, b);
        K6[3] = -newell_nxy(X, Y, Z, a, b, c);
        K6[4] = -newell_nxy(X, Z, Y, a, c, b);
        K6[5] = -newell_nxy(Y, Z, X, b, c, a);
    } else {
        double N6[6];
        gl_far(X, Y, Z, a, b, c, ord, N6);
        for (int q = 0; q < 6; ++q) K6[q] = -N6[q];
    }
    // off-diagonals vanish identically on their odd planes (newell.cpp:201-207)
    if (i == 0 || j == 0) K6[3] = 0.0;
    if (i == 0 || k == 0) K6[4] = 0.0;
    if (j == 0 || k == 0) K6[5] = 0.0;
    for (int q = 0; q < 6; ++q) out[q * n + e] = K6[q];
}

// Transform matrix [H][n]: even -> (d?2:1) cos(2 pi u d/P), odd -> 2 sin(2 pi u d/P) (d>0).
__global__ void k_axis_matrix(int H, int n, int P, int odd, double* __restrict__ C) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)H * n) return;
    const int u = (int)(e / n), d = (int)(e % n);
    const long long m = ((long long)u * d) % P;      // exact argument reduction
    double s, co;
    sincospi(2.0 * (double)m / (double)P, &s, &co);
    C[e] = odd ? (d ? 2.0 * s : 0.0) : (d ? 2.0 * co : 1.0);
}

// K0b: batched fp64 GEMM with arbitrary strides and a two-level batch:
//   out(m,n) = scale * sum_k A(m,k) B(k,n),  batch b = b1*nb2 + b2  (GemmDesc in tensor_api.h).

template <class TO>
__global__ void __launch_bounds__(256) k_gemm64(GemmDesc d, const double* __restrict__ A,
                                                const double* __restrict__ B, TO* __restrict__ O) {
    __shared__ double As[16][65];
    __shared__ double Bs[16][65];
    const int b1 = blockIdx.z / d.nb2, b2 = blockIdx.z % d.nb2;
    A += b1 * d.a_b1 + b2 * d.a_b2;
    B += b1 * d.b_b1 + b2 * d.b_b2;
    O += b1 * d.o_b1 + b2 * d.o_b2;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < d.Kdim; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int kk = e / 64, mm = e % 64;
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < d.Mdim && gk < d.Kdim) ? A[gm * d.a_m + gk * d.a_k] : 0.0;
            const int gn = n0 + mm;
            Bs[kk][mm] = (gn < d.Ndim && gk < d.Kdim) ? B[gk * d.b_k + gn * d.b_n] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = As[kk][ty + 16 * r];
#pragma unroll
            for (int q = 0; q < 4; ++q) bv[q] = Bs[kk][tx + 16 * q];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[r][q] = fma(av[r], bv[q], acc[r][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int gm = m0 + ty + 16 * r, gn = n0 + tx + 16 * q;
            if (gm < d.Mdim && gn < d.Ndim) O[gm * d.o_m + gn * d.o_n] = (TO)(d.scale * acc[r][q]);
        }
}

} // namespace mfd
