/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, called by, or
 * shipped with the product (paper_1406_7459_b200/, include/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * A plain-C restatement of the reference hot path (/root/reference/proj,
 * "magfd"), one translation unit compiled twice: -DORACLE_f64 (REAL=double)
 * and -DORACLE_f32 (REAL=float), mirroring the reference's template on T.
 * It follows the reference operation order so that its f64 results can be
 * pinned bitwise against oracle/_ref (the reference itself) on small grids,
 * and against the 12 Maple Newell goldens (proj/tests/test_demag.cpp:26-44).
 *
 *   orc_nxx / orc_nxy / orc_tensor_entry  newell.cpp:14-209 (long double)
 *   padded sizes, wrap layout             demag.hpp:24-37, 49-90
 *   radix-2 FFT (bit reversal + DIT)      fft.hpp:58-116, 164-237
 *   spectral multiply                     demag.hpp:150-171
 *   demag pipeline                        demag.hpp:194-251
 *   exchange / anisotropy / Zeeman        fields.hpp:21-81, 220-253
 *   LLG rhs / max torque / Euler          dynamics.hpp:49-121
 *   Simulation::step                      sim.hpp:33-42
 *   reducedMean                           state.hpp:113-124
 *   energies                              fields.hpp:127-190
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#if defined(ORACLE_f32)
typedef float REAL;
#define SFX(n) n##_f32
#define RSQRT sqrtf
#else
typedef double REAL;
#define SFX(n) n##_f64
#define RSQRT sqrt
#endif

typedef long double LD;
static const LD PI_LD = 3.14159265358979323846264338327950288L;
static const double PI_D = 3.14159265358979323846;
static const double MU0 = 4.0e-7 * 3.14159265358979323846;

/* ---------------------------------------------------------------- Newell */

/* Neumaier compensated sum (newell.cpp:14-26). */
static LD csum(const LD* v, int n) {
    LD s = v[0], c = 0.0L;
    for (int i = 1; i < n; ++i) {
        LD t = s + v[i];
        c += fabsl(s) >= fabsl(v[i]) ? (s - t) + v[i] : (v[i] - t) + s;
        s = t;
    }
    return s + c;
}

/* Self factor of one prism (newell.cpp:31-58). */
static LD self_nx(LD x, LD y, LD z) {
    if (x <= 0 || y <= 0 || z <= 0) return 0;
    if (x == y && y == z) return 1.0L / 3.0L;
    LD x2 = x * x, y2 = y * y, z2 = z * z, R = sqrtl(x2 + y2 + z2);
    LD dxy = (x - y) * (x + y), dxz = (x - z) * (x + z);
    LD a[15];
    a[0] = -4.0L * (2.0L * x2 * x - y2 * y - z2 * z);
    a[1] = 4.0L * (x2 + dxy) * sqrtl(x2 + y2);
    a[2] = 4.0L * (x2 + dxz) * sqrtl(x2 + z2);
    a[3] = -4.0L * (y2 + z2) * sqrtl(y2 + z2);
    a[4] = -4.0L * R * (dxy + dxz);
    a[5] = 24.0L * x * y * z * atanl(y * z / (x * R));
    a[6] = 12.0L * (z + y) * x2 * logl(x);
    a[7] = 12.0L * z * y2 * logl((sqrtl(y2 + z2) + z) / y);
    a[8] = -12.0L * z * x2 * logl(sqrtl(x2 + z2) + z);
    a[9] = 12.0L * z * dxy * logl(R + z);
    a[10] = -6.0L * z * dxy * logl(x2 + y2);
    a[11] = 12.0L * y * z2 * logl((sqrtl(y2 + z2) + y) / z);
    a[12] = -12.0L * y * x2 * logl(sqrtl(x2 + y2) + y);
    a[13] = 12.0L * y * dxz * logl(R + y);
    a[14] = -6.0L * y * dxz * logl(x2 + z2);
    return csum(a, 15) / (12.0L * PI_LD * x * y * z);
}

/* Newell f (newell.cpp:61-98). */
static LD nf(LD x, LD y, LD z) {
    x = fabsl(x); y = fabsl(y); z = fabsl(z);
    LD x2 = x * x, y2 = y * y, z2 = z * z, r = x2 + y2 + z2;
    if (r <= 0) return 0;
    r = sqrtl(r);
    LD p[8];
    int n = 0;
    if (z > 0) {
        p[n++] = 2.0L * (2.0L * x2 - y2 - z2) * r;
        if (x > 0 && y > 0) p[n++] = -12.0L * x * y * z * atan2l(y * z, x * r);
        if (y > 0 && x2 + z2 > 0) {
            LD l = logl(((y + r) * (y + r)) / (x2 + z2));
            p[n++] = 3.0L * y * z2 * l;
            p[n++] = -3.0L * y * x2 * l;
        }
        if (x2 + y2 > 0) {
            LD l = logl(((z + r) * (z + r)) / (x2 + y2));
            p[n++] = 3.0L * z * y2 * l;
            p[n++] = -3.0L * z * x2 * l;
        }
    } else if (x == y) {
        p[n++] = -2.4598143973710680537922785014593576970294L * x2 * x;
    } else {
        p[n++] = 2.0L * (2.0L * x2 - y2) * r;
        if (y > 0 && x > 0) p[n++] = -6.0L * y * x2 * logl((y + r) / x);
    }
    return csum(p, n) / 12.0L;
}

/* Newell g (newell.cpp:101-132). */
static LD ng(LD x, LD y, LD z) {
    LD sg = 1;
    if (x < 0) sg = -sg;
    if (y < 0) sg = -sg;
    x = fabsl(x); y = fabsl(y); z = fabsl(z);
    LD x2 = x * x, y2 = y * y, z2 = z * z, r = x2 + y2 + z2;
    if (r <= 0) return 0;
    r = sqrtl(r);
    LD p[7];
    int n = 0;
    p[n++] = -2.0L * x * y * r;
    if (z > 0) {
        p[n++] = -z * z2 * atan2l(x * y, z * r);
        p[n++] = -3.0L * z * y2 * atan2l(x * z, y * r);
        p[n++] = -3.0L * z * x2 * atan2l(y * z, x * r);
        if (x2 + y2 > 0) p[n++] = 6.0L * x * y * z * logl((z + r) / sqrtl(x2 + y2));
        if (y2 + z2 > 0) p[n++] = y * (3.0L * z2 - y2) * logl((x + r) / sqrtl(y2 + z2));
        if (x2 + z2 > 0) p[n++] = x * (3.0L * z2 - x2) * logl((y + r) / sqrtl(x2 + z2));
    } else {
        if (y > 0) p[n++] = -y * y2 * logl((x + r) / y);
        if (x > 0) p[n++] = -x * x2 * logl((y + r) / x);
    }
    return sg * csum(p, n) / 6.0L;
}

/* 27-point second difference in the reference's term order (newell.cpp:138-173). */
static LD stencil27(LD (*f)(LD, LD, LD), LD x, LD y, LD z, LD a, LD b, LD c) {
    static const signed char off[27][4] = {
        {1, 1, 1, -1},  {1, -1, 1, -1}, {1, -1, -1, -1}, {1, 1, -1, -1}, {-1, 1, -1, -1},
        {-1, 1, 1, -1}, {-1, -1, 1, -1}, {-1, -1, -1, -1}, {0, -1, -1, 2}, {0, -1, 1, 2},
        {0, 1, 1, 2},   {0, 1, -1, 2},  {1, 1, 0, 2},    {1, 0, 1, 2},    {1, 0, -1, 2},
        {1, -1, 0, 2},  {-1, -1, 0, 2}, {-1, 0, 1, 2},   {-1, 0, -1, 2},  {-1, 1, 0, 2},
        {0, -1, 0, -4}, {0, 1, 0, -4},  {0, 0, -1, -4},  {0, 0, 1, -4},   {1, 0, 0, -4},
        {-1, 0, 0, -4}, {0, 0, 0, 8}};
    LD v[27];
    for (int t = 0; t < 27; ++t) {
        LD px = off[t][0] > 0 ? x + a : off[t][0] < 0 ? x - a : x;
        LD py = off[t][1] > 0 ? y + b : off[t][1] < 0 ? y - b : y;
        LD pz = off[t][2] > 0 ? z + c : off[t][2] < 0 ? z - c : z;
        v[t] = (LD)off[t][3] * f(px, py, pz);
    }
    return csum(v, 27);
}

double SFX(orc_nxx)(double X, double Y, double Z, double a, double b, double c) {
    if (X == 0 && Y == 0 && Z == 0) return (double)self_nx(a, b, c);
    return (double)(stencil27(nf, X, Y, Z, a, b, c) / (4.0L * PI_LD * (LD)a * (LD)b * (LD)c));
}
double SFX(orc_nxy)(double X, double Y, double Z, double a, double b, double c) {
    return (double)(stencil27(ng, X, Y, Z, a, b, c) / (4.0L * PI_LD * (LD)a * (LD)b * (LD)c));
}
static LD nxx_ld(LD X, LD Y, LD Z, LD a, LD b, LD c) {
    if (X == 0 && Y == 0 && Z == 0) return self_nx(a, b, c);
    return stencil27(nf, X, Y, Z, a, b, c) / (4.0L * PI_LD * a * b * c);
}
static LD nxy_ld(LD X, LD Y, LD Z, LD a, LD b, LD c) {
    return stencil27(ng, X, Y, Z, a, b, c) / (4.0L * PI_LD * a * b * c);
}

/* K = -N with parity signs (newell.cpp:188-209); out = xx,yy,zz,xy,xz,yz. */
void SFX(orc_tensor_entry)(int di, int dj, int dk, double dx, double dy, double dz,
                           double out[6]) {
    int ai = abs(di), aj = abs(dj), ak = abs(dk);
    LD X = ai * (LD)dx, Y = aj * (LD)dy, Z = ak * (LD)dz;
    out[0] = (double)(-nxx_ld(X, Y, Z, dx, dy, dz));
    out[1] = (double)(-nxx_ld(Y, Z, X, dy, dz, dx));
    out[2] = (double)(-nxx_ld(Z, X, Y, dz, dx, dy));
    int sx = di < 0 ? -1 : 1, sy = dj < 0 ? -1 : 1, sz = dk < 0 ? -1 : 1;
    out[3] = out[4] = out[5] = 0.0;
    if (ai && aj) out[3] = sx * sy * (double)(-nxy_ld(X, Y, Z, dx, dy, dz));
    if (ai && ak) out[4] = sx * sz * (double)(-nxy_ld(X, Z, Y, dx, dz, dy));
    if (aj && ak) out[5] = sy * sz * (double)(-nxy_ld(Y, Z, X, dy, dz, dx));
}

/* ------------------------------------------------------------------- FFT */

typedef struct { REAL re, im; } cplx;

static int next_pow2(int n) { int p = 1; while (p < n) p <<= 1; return p; }
static int padded(int n) { return next_pow2(2 * n); } /* demag.hpp:24 */

typedef struct { int n; int* rev; cplx* tw; } line_t;

static void line_init(line_t* L, int n) {
    int bits = 0;
    L->n = n;
    while ((1 << bits) < n) ++bits;
    L->rev = malloc(sizeof(int) * n);
    for (int i = 0; i < n; ++i) {
        int r = 0;
        for (int b = 0; b < bits; ++b) if (i & (1 << b)) r |= 1 << (bits - 1 - b);
        L->rev[i] = r;
    }
    L->tw = malloc(sizeof(cplx) * (n / 2 > 0 ? n / 2 : 1));
    for (int k = 0; k < n / 2; ++k) {   /* long-double tables cast to REAL (fft.hpp:70-74) */
        LD a = -2.0L * (LD)PI_D * k / n;
        L->tw[k].re = (REAL)cosl(a);
        L->tw[k].im = (REAL)sinl(a);
    }
}
static void line_free(line_t* L) { free(L->rev); free(L->tw); }

/* In-place radix-2 over n rows at stride rs, columns [lo,hi) (fft.hpp:92-116). */
static void rows(const line_t* L, cplx* base, size_t rs, size_t lo, size_t hi, int inv) {
    int n = L->n;
    for (int j = 0; j < n; ++j)
        if (L->rev[j] > j)
            for (size_t c = lo; c < hi; ++c) {
                cplx t = base[j * rs + c];
                base[j * rs + c] = base[(size_t)L->rev[j] * rs + c];
                base[(size_t)L->rev[j] * rs + c] = t;
            }
    for (int len = 2; len <= n; len <<= 1) {
        int half = len >> 1, st = n / len;
        for (int rb = 0; rb < n; rb += len)
            for (int j = 0; j < half; ++j) {
                cplx w = L->tw[j * st];
                if (inv) w.im = -w.im;
                cplx* a = base + (size_t)(rb + j) * rs;
                cplx* b = base + (size_t)(rb + j + half) * rs;
                for (size_t c = lo; c < hi; ++c) {
                    cplx u = a[c], v;
                    v.re = b[c].re * w.re - b[c].im * w.im;
                    v.im = b[c].re * w.im + b[c].im * w.re;
                    a[c].re = u.re + v.re; a[c].im = u.im + v.im;
                    b[c].re = u.re - v.re; b[c].im = u.im - v.im;
                }
            }
    }
}

typedef struct { int px, py, pz; line_t lx, ly, lz; } plan_t;

static void fft3(const plan_t* p, cplx* d, int inv, int ay, int az) {
    size_t plane = (size_t)p->px * p->py;
    if (!inv) { /* forwardPadded: x over active rows, y over active planes, z (fft.hpp:173-178) */
        for (int k = 0; k < az; ++k)
            for (int j = 0; j < ay; ++j) rows(&p->lx, d + ((size_t)j + (size_t)p->py * k) * p->px, 1, 0, 1, 0);
        for (int k = 0; k < az; ++k) rows(&p->ly, d + k * plane, p->px, 0, p->px, 0);
        rows(&p->lz, d, plane, 0, plane, 0);
    } else {    /* inverseCorner: z, y (needed planes), x (needed rows) (fft.hpp:181-186) */
        rows(&p->lz, d, plane, 0, plane, 1);
        for (int k = 0; k < az; ++k) rows(&p->ly, d + k * plane, p->px, 0, p->px, 1);
        for (int k = 0; k < az; ++k)
            for (int j = 0; j < ay; ++j) rows(&p->lx, d + ((size_t)j + (size_t)p->py * k) * p->px, 1, 0, 1, 1);
    }
}

/* rows() with rs=1 and columns [0,1) transforms one contiguous line. */

/* ------------------------------------------------------------- context */

typedef struct {
    int nx, ny, nz;
    double dx, dy, dz;
    double A, Ku, Ms, alpha, gamma;
    double easy_axis[3];
    int exchange, anisotropy, demag, zeeman;
    double h_ext[3];
    double dt;
    int renorm_every;
} orc_spec;

typedef struct {
    orc_spec s;
    size_t n;
    plan_t plan;
    cplx* K[6];        /* full complex tensor spectra (demag.hpp:105-119) */
    cplx* w[3];        /* scratch lattices */
    REAL *mx, *my, *mz, *hx, *hy, *hz, *dxh, *dyh, *dzh;
    double t;
    long step;
} orc_ctx;

void* SFX(orc_create)(const orc_spec* s) {
    orc_ctx* c = calloc(1, sizeof(orc_ctx));
    c->s = *s;
    c->n = (size_t)s->nx * s->ny * s->nz;
    REAL** f[] = {&c->mx, &c->my, &c->mz, &c->hx, &c->hy, &c->hz, &c->dxh, &c->dyh, &c->dzh};
    for (int i = 0; i < 9; ++i) *f[i] = calloc(c->n, sizeof(REAL));
    if (s->demag) {
        plan_t* p = &c->plan;
        p->px = padded(s->nx); p->py = padded(s->ny); p->pz = padded(s->nz);
        line_init(&p->lx, p->px); line_init(&p->ly, p->py); line_init(&p->lz, p->pz);
        size_t P = (size_t)p->px * p->py * p->pz;
        for (int q = 0; q < 6; ++q) c->K[q] = calloc(P, sizeof(cplx));
        for (int q = 0; q < 3; ++q) c->w[q] = calloc(P, sizeof(cplx));
        /* buildDemagTensor: octant evaluation mirrored with parity signs (demag.hpp:66-88) */
        for (int k = 0; k < s->nz; ++k)
            for (int j = 0; j < s->ny; ++j)
                for (int i = 0; i < s->nx; ++i) {
                    double e[6];
                    SFX(orc_tensor_entry)(i, j, k, s->dx, s->dy, s->dz, e);
                    for (int sx = 0; sx < (i > 0 ? 2 : 1); ++sx)
                        for (int sy = 0; sy < (j > 0 ? 2 : 1); ++sy)
                            for (int sz = 0; sz < (k > 0 ? 2 : 1); ++sz) {
                                int wi = sx ? p->px - i : i, wj = sy ? p->py - j : j,
                                    wk = sz ? p->pz - k : k;
                                size_t slot = wi + (size_t)p->px * (wj + (size_t)p->py * wk);
                                double ox = sx ? -1.0 : 1.0, oy = sy ? -1.0 : 1.0,
                                       oz = sz ? -1.0 : 1.0;
                                c->K[0][slot].re = (REAL)e[0];
                                c->K[1][slot].re = (REAL)e[1];
                                c->K[2][slot].re = (REAL)e[2];
                                c->K[3][slot].re = (REAL)(ox * oy * e[3]);
                                c->K[4][slot].re = (REAL)(ox * oz * e[4]);
                                c->K[5][slot].re = (REAL)(oy * oz * e[5]);
                            }
                }
        for (int q = 0; q < 6; ++q) fft3(p, c->K[q], 0, p->py, p->pz);
    }
    return c;
}

void SFX(orc_destroy)(void* h) {
    orc_ctx* c = h;
    if (!c) return;
    REAL* f[] = {c->mx, c->my, c->mz, c->hx, c->hy, c->hz, c->dxh, c->dyh, c->dzh};
    for (int i = 0; i < 9; ++i) free(f[i]);
    if (c->s.demag) {
        for (int q = 0; q < 6; ++q) free(c->K[q]);
        for (int q = 0; q < 3; ++q) free(c->w[q]);
        line_free(&c->plan.lx); line_free(&c->plan.ly); line_free(&c->plan.lz);
    }
    free(c);
}

void SFX(orc_set_m)(void* h, const double* x, const double* y, const double* z) {
    orc_ctx* c = h;
    for (size_t i = 0; i < c->n; ++i) { c->mx[i] = (REAL)x[i]; c->my[i] = (REAL)y[i]; c->mz[i] = (REAL)z[i]; }
}
void SFX(orc_get_m)(void* h, double* x, double* y, double* z) {
    orc_ctx* c = h;
    for (size_t i = 0; i < c->n; ++i) { x[i] = c->mx[i]; y[i] = c->my[i]; z[i] = c->mz[i]; }
}
void SFX(orc_set_time)(void* h, double t, long step) { orc_ctx* c = h; c->t = t; c->step = step; }
void SFX(orc_get_time)(void* h, double* t, long* step) { orc_ctx* c = h; *t = c->t; *step = c->step; }

/* DemagConvolution::field (demag.hpp:194-251) into c->dxh/dyh/dzh. */
static void demag_field(orc_ctx* c) {
    const plan_t* p = &c->plan;
    const orc_spec* s = &c->s;
    size_t P = (size_t)p->px * p->py * p->pz, px = p->px, pxy = (size_t)p->px * p->py;
    const REAL* src[3] = {c->mx, c->my, c->mz};
    for (int q = 0; q < 3; ++q) {
        memset(c->w[q], 0, P * sizeof(cplx));
        for (int k = 0; k < s->nz; ++k)
            for (int j = 0; j < s->ny; ++j)
                for (int i = 0; i < s->nx; ++i) {
                    size_t cell = i + (size_t)s->nx * (j + (size_t)s->ny * k);
                    c->w[q][i + px * j + pxy * k].re = src[q][cell];
                }
        fft3(p, c->w[q], 0, s->ny, s->nz);
    }
    /* spectralMultiply: symmetric complex 3x3 per bin (demag.hpp:165-170) */
    for (size_t b = 0; b < P; ++b) {
        cplx x = c->w[0][b], y = c->w[1][b], z = c->w[2][b];
        const cplx *kxx = &c->K[0][b], *kyy = &c->K[1][b], *kzz = &c->K[2][b],
                   *kxy = &c->K[3][b], *kxz = &c->K[4][b], *kyz = &c->K[5][b];
#define CM(a, k) ((cplx){(a).re * (k)->re - (a).im * (k)->im, (a).re * (k)->im + (a).im * (k)->re})
        cplx t1 = CM(x, kxx), t2 = CM(y, kxy), t3 = CM(z, kxz);
        c->w[0][b] = (cplx){t1.re + t2.re + t3.re, t1.im + t2.im + t3.im};
        t1 = CM(x, kxy); t2 = CM(y, kyy); t3 = CM(z, kyz);
        c->w[1][b] = (cplx){t1.re + t2.re + t3.re, t1.im + t2.im + t3.im};
        t1 = CM(x, kxz); t2 = CM(y, kyz); t3 = CM(z, kzz);
        c->w[2][b] = (cplx){t1.re + t2.re + t3.re, t1.im + t2.im + t3.im};
#undef CM
    }
    REAL* dst[3] = {c->dxh, c->dyh, c->dzh};
    const REAL scale = (REAL)(1.0 / (double)P);
    for (int q = 0; q < 3; ++q) {
        fft3(p, c->w[q], 1, s->ny, s->nz);
        for (int k = 0; k < s->nz; ++k)
            for (int j = 0; j < s->ny; ++j)
                for (int i = 0; i < s->nx; ++i)
                    dst[q][i + (size_t)s->nx * (j + (size_t)s->ny * k)] =
                        c->w[q][i + px * j + pxy * k].re * scale;
    }
}

/* EffectiveFieldProvider::compute (fields.hpp:220-253) into c->hx/hy/hz. */
static void heff(orc_ctx* c) {
    const orc_spec* s = &c->s;
    size_t n = c->n;
    if (s->demag) {
        demag_field(c);
        memcpy(c->hx, c->dxh, n * sizeof(REAL));
        memcpy(c->hy, c->dyh, n * sizeof(REAL));
        memcpy(c->hz, c->dzh, n * sizeof(REAL));
    } else {
        memset(c->hx, 0, n * sizeof(REAL)); memset(c->hy, 0, n * sizeof(REAL)); memset(c->hz, 0, n * sizeof(REAL));
    }
    if (s->exchange && s->A > 0) { /* fields.hpp:21-53 */
        double base = 2.0 * s->A / (MU0 * s->Ms * s->Ms);
        REAL cx = (REAL)(base / (s->dx * s->dx)), cy = (REAL)(base / (s->dy * s->dy)),
             cz = (REAL)(base / (s->dz * s->dz));
        size_t sy = s->nx, sz = (size_t)s->nx * s->ny;
        for (int k = 0; k < s->nz; ++k)
            for (int j = 0; j < s->ny; ++j)
                for (int i = 0; i < s->nx; ++i) {
                    size_t q = i + sy * j + sz * k;
                    REAL h0 = 0, h1 = 0, h2 = 0;
#define ADD(nb, w) { h0 += (w) * (c->mx[nb] - c->mx[q]); h1 += (w) * (c->my[nb] - c->my[q]); h2 += (w) * (c->mz[nb] - c->mz[q]); }
                    if (i > 0) ADD(q - 1, cx);
                    if (i < s->nx - 1) ADD(q + 1, cx);
                    if (j > 0) ADD(q - sy, cy);
                    if (j < s->ny - 1) ADD(q + sy, cy);
                    if (k > 0) ADD(q - sz, cz);
                    if (k < s->nz - 1) ADD(q + sz, cz);
#undef ADD
                    c->hx[q] += h0; c->hy[q] += h1; c->hz[q] += h2;
                }
    }
    if (s->anisotropy && s->Ku != 0) { /* fields.hpp:66-81 */
        REAL cc = (REAL)(2.0 * s->Ku / (MU0 * s->Ms * s->Ms));
        REAL a0 = (REAL)s->easy_axis[0], a1 = (REAL)s->easy_axis[1], a2 = (REAL)s->easy_axis[2];
        for (size_t q = 0; q < n; ++q) {
            REAL proj = cc * (c->mx[q] * a0 + c->my[q] * a1 + c->mz[q] * a2);
            c->hx[q] += proj * a0; c->hy[q] += proj * a1; c->hz[q] += proj * a2;
        }
    }
    if (s->zeeman) { /* fields.hpp:243-251 */
        REAL e0 = (REAL)s->h_ext[0], e1 = (REAL)s->h_ext[1], e2 = (REAL)s->h_ext[2];
        if (e0 != 0 || e1 != 0 || e2 != 0)
            for (size_t q = 0; q < n; ++q) { c->hx[q] += e0; c->hy[q] += e1; c->hz[q] += e2; }
    }
}

void SFX(orc_heff)(void* h, double* x, double* y, double* z) {
    orc_ctx* c = h;
    heff(c);
    for (size_t i = 0; i < c->n; ++i) { x[i] = c->hx[i]; y[i] = c->hy[i]; z[i] = c->hz[i]; }
}
int SFX(orc_hdemag)(void* h, double* x, double* y, double* z) {
    orc_ctx* c = h;
    if (!c->s.demag) return 3; /* logic_error (fields.hpp:264-267) */
    heff(c);
    for (size_t i = 0; i < c->n; ++i) { x[i] = c->dxh[i]; y[i] = c->dyh[i]; z[i] = c->dzh[i]; }
    return 0;
}

/* Simulation::step x n (sim.hpp:33-42); torques[i] = pre-step max torque of
 * step i in deg/ns.  Returns 2 on a non-finite update (dynamics.hpp:115-117). */
int SFX(orc_step)(void* h, long nsteps, double* torques) {
    orc_ctx* c = h;
    const orc_spec* s = &c->s;
    size_t n = c->n;
    const double a2 = 1.0 + s->alpha * s->alpha;
    const REAL prec = (REAL)(-s->gamma / a2), damp = (REAL)(-s->alpha * s->gamma / (a2 * s->Ms));
    const REAL mu0 = (REAL)MU0, dtT = (REAL)s->dt, msT = (REAL)s->Ms;
    REAL* r[3];
    for (int q = 0; q < 3; ++q) r[q] = malloc(n * sizeof(REAL));
    int rc = 0;
    for (long it = 0; it < nsteps; ++it) {
        heff(c);
        double mx2 = -1;
        for (size_t q = 0; q < n; ++q) { /* llgRhs (dynamics.hpp:58-63) */
            REAL m0 = c->mx[q], m1 = c->my[q], m2 = c->mz[q];
            REAL h0 = mu0 * c->hx[q], h1 = mu0 * c->hy[q], h2 = mu0 * c->hz[q];
            REAL c0 = m1 * h2 - m2 * h1, c1 = m2 * h0 - m0 * h2, c2 = m0 * h1 - m1 * h0;
            REAL d0 = m1 * c2 - m2 * c1, d1 = m2 * c0 - m0 * c2, d2 = m0 * c1 - m1 * c0;
            r[0][q] = prec * c0 + damp * d0;
            r[1][q] = prec * c1 + damp * d1;
            r[2][q] = prec * c2 + damp * d2;
            double v0 = r[0][q], v1 = r[1][q], v2 = r[2][q];
            double t2 = v0 * v0 + v1 * v1 + v2 * v2;    /* maxTorqueRate (dynamics.hpp:76-81) */
            if (q == 0 || t2 > mx2) mx2 = t2;
        }
        if (torques) torques[it] = sqrt(mx2) / s->Ms * (180.0 / PI_D * 1e-9);
        int renorm = (c->step + 1) % s->renorm_every == 0;
        int bad = 0;
        for (size_t q = 0; q < n; ++q) { /* eulerUpdate (dynamics.hpp:100-114) */
            REAL m0 = c->mx[q] + dtT * r[0][q], m1 = c->my[q] + dtT * r[1][q],
                 m2 = c->mz[q] + dtT * r[2][q];
            if (renorm) {
                REAL n2 = m0 * m0 + m1 * m1 + m2 * m2;
                if (!(n2 > 0) || !isfinite((double)n2)) { bad = 1; continue; }
                REAL f = msT / RSQRT(n2);
                m0 = f * m0; m1 = f * m1; m2 = f * m2;
            } else if (!isfinite((double)(m0 + m1 + m2))) { bad = 1; continue; }
            c->mx[q] = m0; c->my[q] = m1; c->mz[q] = m2;
        }
        if (bad) { rc = 2; break; }
        c->t += s->dt;
        c->step += 1;
    }
    for (int q = 0; q < 3; ++q) free(r[q]);
    return rc;
}

/* reducedMean (state.hpp:113-124): serial double sum. */
void SFX(orc_reduced_mean)(void* h, double m[3]) {
    orc_ctx* c = h;
    double sx = 0, sy = 0, sz = 0;
    for (size_t q = 0; q < c->n; ++q) { sx += c->mx[q]; sy += c->my[q]; sz += c->mz[q]; }
    double sc = 1.0 / (c->s.Ms * (double)c->n);
    m[0] = sx * sc; m[1] = sy * sc; m[2] = sz * sc;
}

/* energies (fields.hpp:127-190, serial ordering) of the current M using a
 * fresh field evaluation; out = exch, anis, demag, zeeman, total. */
void SFX(orc_energies)(void* h, double out[5]) {
    orc_ctx* c = h;
    const orc_spec* s = &c->s;
    heff(c);
    double V = s->dx * s->dy * s->dz, ex = 0, an = 0, de = 0, ze = 0;
    size_t sy = s->nx, sz = (size_t)s->nx * s->ny;
    if (s->exchange && s->A > 0) {
        double wx = 1.0 / (s->dx * s->dx), wy = 1.0 / (s->dy * s->dy), wz = 1.0 / (s->dz * s->dz);
        for (int k = 0; k < s->nz; ++k)
            for (int j = 0; j < s->ny; ++j)
                for (int i = 0; i < s->nx; ++i) {
                    size_t q = i + sy * j + sz * k;
                    double acc = 0;
#define LINK(nb, w) { double e0 = (double)c->mx[nb] - c->mx[q], e1 = (double)c->my[nb] - c->my[q], e2 = (double)c->mz[nb] - c->mz[q]; acc += (w) * (e0 * e0 + e1 * e1 + e2 * e2); }
                    if (i < s->nx - 1) LINK(q + 1, wx);
                    if (j < s->ny - 1) LINK(q + sy, wy);
                    if (k < s->nz - 1) LINK(q + sz, wz);
#undef LINK
                    ex += acc;
                }
        ex *= s->A * V / (s->Ms * s->Ms);
    }
    if (s->anisotropy && s->Ku != 0) {
        for (size_t q = 0; q < c->n; ++q) {
            double m0 = (double)c->mx[q] / s->Ms, m1 = (double)c->my[q] / s->Ms, m2 = (double)c->mz[q] / s->Ms;
            double p = m0 * s->easy_axis[0] + m1 * s->easy_axis[1] + m2 * s->easy_axis[2];
            an += 1.0 - p * p;
        }
        an *= s->Ku * V;
    }
    if (s->demag) {
        for (size_t q = 0; q < c->n; ++q)
            de += (double)c->dxh[q] * c->mx[q] + (double)c->dyh[q] * c->my[q] + (double)c->dzh[q] * c->mz[q];
        de *= -0.5 * MU0 * V;
    }
    if (s->zeeman && (s->h_ext[0] != 0 || s->h_ext[1] != 0 || s->h_ext[2] != 0)) {
        for (size_t q = 0; q < c->n; ++q)
            ze += s->h_ext[0] * c->mx[q] + s->h_ext[1] * c->my[q] + s->h_ext[2] * c->mz[q];
        ze *= -MU0 * V;
    }
    out[0] = ex; out[1] = an; out[2] = de; out[3] = ze; out[4] = ex + an + de + ze;
}

/* Direct long-double demag sum (oracle.hpp:26-70), grid-size capped by caller. */
void SFX(orc_direct_demag)(int nx, int ny, int nz, double dx, double dy, double dz,
                           const double* mx, const double* my, const double* mz,
                           double* hx, double* hy, double* hz) {
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                LD a0 = 0, a1 = 0, a2 = 0;
                for (int n = 0; n < nz; ++n)
                    for (int m = 0; m < ny; ++m)
                        for (int l = 0; l < nx; ++l) {
                            double e[6];
                            size_t src = l + (size_t)nx * (m + (size_t)ny * n);
                            SFX(orc_tensor_entry)(l - i, m - j, n - k, dx, dy, dz, e);
                            LD x = mx[src], y = my[src], z = mz[src];
                            a0 += x * e[0] + y * e[3] + z * e[4];
                            a1 += x * e[3] + y * e[1] + z * e[5];
                            a2 += x * e[4] + y * e[5] + z * e[2];
                        }
                size_t c = i + (size_t)nx * (j + (size_t)ny * k);
                hx[c] = (double)a0; hy[c] = (double)a1; hz[c] = (double)a2;
            }
}
