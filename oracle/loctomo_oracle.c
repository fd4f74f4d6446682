/*
 * loctomo_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * local approximation of regularized iterative tomography
 * (Pelt & Batenburg, arXiv 1604.02292; PAPER.md in the task's reference).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_1604_02292_b200/) never includes, links or calls it,
 * and this file includes nothing from the product.
 *
 * Every function cites the PAPER.md passage ("P:Lnnn") it follows and the
 * DESIGN.md reading (A*) it takes where the paper is silent.
 *
 * Conventions (V1/V2, reading A1/A2):
 *   pixel (i,j): row i (top = 0), column j; centre x_j = j-(N-1)/2,
 *   y_i = (N-1)/2 - i; detector bin d has centre t_d = d-(N_d-1)/2;
 *   W[(a,d),(i,j)] = (1/c_a) * hat((t_d - (x_j cos th_a + y_i sin th_a))/c_a),
 *   c_a = max(|cos th_a|, |sin th_a|), hat(u) = max(0, 1-|u|)
 *   (Joseph's ray-driven interpolation written as the closed-form matrix
 *   element; tests/test_oracle_pins.py pins it against explicit ray marching).
 *
 * OpenMP parallelism only over independent outputs (sinogram rows, image
 * rows, ROIs); every output element is summed by one thread in a fixed
 * order, so results do not depend on the thread count.  Built without
 * -ffast-math.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_RUNTIME 1
#define OR_ERR_INVALID 2

static double hat(double u) {
    double a = fabs(u);
    return a < 1.0 ? 1.0 - a : 0.0;
}

void or_set_threads(int nt) {
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
#else
    (void)nt;
#endif
}

int or_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Projector on a rectangle of pixels.  img points at pixel (r0, c0) of an
 * image with row stride `stride`; the rectangle is h x w pixels.
 * P:L244 (W: discretized line integrals; W^T its transpose),
 * P:L250-251 (W_L = W M_L, W_L^T = M_L W^T): restricting the loops to the
 * pixels of L is exactly multiplication by the mask M_L.
 * ------------------------------------------------------------------------- */

/* sino[a*nd + d] += sum_{(i,j) in rect} W[(a,d),(i,j)] img(i,j); sino is zeroed first. */
static void fp_rect(int n, int na, int nd, const double* ang,
                    const double* img, int stride, int r0, int c0, int h, int w,
                    double* sino) {
    const double half_n = 0.5 * (n - 1), half_d = 0.5 * (nd - 1);
#pragma omp parallel for schedule(static)
    for (int a = 0; a < na; ++a) {
        const double cs = cos(ang[a]), sn = sin(ang[a]);
        const double c = fmax(fabs(cs), fabs(sn));
        double* row = sino + (size_t)a * nd;
        for (int d = 0; d < nd; ++d) row[d] = 0.0;
        for (int i = 0; i < h; ++i) {
            const double y = half_n - (r0 + i);
            for (int j = 0; j < w; ++j) {
                const double v = img[(size_t)i * stride + j];
                if (v == 0.0) continue;
                const double x = (c0 + j) - half_n;
                const double tau = x * cs + y * sn + half_d; /* bin coordinate of the pixel centre */
                int dlo = (int)floor(tau - c), dhi = (int)ceil(tau + c);
                if (dlo < 0) dlo = 0;
                if (dhi > nd - 1) dhi = nd - 1;
                for (int d = dlo; d <= dhi; ++d) row[d] += hat((d - tau) / c) / c * v;
            }
        }
    }
}

/* img(i,j) = sum_a sum_d W[(a,d),(i,j)] sino[a][d] for (i,j) in the rect. */
static void bp_rect(int n, int na, int nd, const double* ang, const double* sino,
                    double* img, int stride, int r0, int c0, int h, int w) {
    const double half_n = 0.5 * (n - 1), half_d = 0.5 * (nd - 1);
    double* cs = (double*)malloc(sizeof(double) * na * 3);
    for (int a = 0; a < na; ++a) {
        cs[3 * a] = cos(ang[a]);
        cs[3 * a + 1] = sin(ang[a]);
        cs[3 * a + 2] = fmax(fabs(cs[3 * a]), fabs(cs[3 * a + 1]));
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < h; ++i) {
        const double y = half_n - (r0 + i);
        for (int j = 0; j < w; ++j) {
            const double x = (c0 + j) - half_n;
            double acc = 0.0;
            for (int a = 0; a < na; ++a) {
                const double c = cs[3 * a + 2];
                const double tau = x * cs[3 * a] + y * cs[3 * a + 1] + half_d;
                int dlo = (int)floor(tau - c), dhi = (int)ceil(tau + c);
                if (dlo < 0) dlo = 0;
                if (dhi > nd - 1) dhi = nd - 1;
                const double* row = sino + (size_t)a * nd;
                for (int d = dlo; d <= dhi; ++d) acc += hat((d - tau) / c) / c * row[d];
            }
            img[(size_t)i * stride + j] = acc;
        }
    }
    free(cs);
}

static int check_geom(int n, int na, int nd, const double* ang) {
    if (n < 1 || na < 1 || nd < 1 || !ang) return OR_ERR_INVALID;
    for (int a = 0; a < na; ++a) {
        if (!(ang[a] >= 0.0 && ang[a] < M_PI)) return OR_ERR_INVALID;
        if (a && !(ang[a] > ang[a - 1])) return OR_ERR_INVALID;
    }
    return OR_OK;
}

/* W M_R x for the rect R = [r0,r1) x [c0,c1) of a full N x N image. */
int or_forward(int n, int na, int nd, const double* ang, const double* img,
               int r0, int r1, int c0, int c1, double* sino) {
    if (check_geom(n, na, nd, ang)) return OR_ERR_INVALID;
    if (r0 < 0 || c0 < 0 || r1 > n || c1 > n || r0 > r1 || c0 > c1) return OR_ERR_INVALID;
    fp_rect(n, na, nd, ang, img + (size_t)r0 * n + c0, n, r0, c0, r1 - r0, c1 - c0, sino);
    return OR_OK;
}

/* M_R W^T s on a full N x N image (zero outside R). */
int or_back(int n, int na, int nd, const double* ang, const double* sino,
            int r0, int r1, int c0, int c1, double* img) {
    if (check_geom(n, na, nd, ang)) return OR_ERR_INVALID;
    if (r0 < 0 || c0 < 0 || r1 > n || c1 > n || r0 > r1 || c0 > c1) return OR_ERR_INVALID;
    memset(img, 0, sizeof(double) * (size_t)n * n);
    bp_rect(n, na, nd, ang, sino, img + (size_t)r0 * n + c0, n, r0, c0, r1 - r0, c1 - c0);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Alg. 1 (alg:filtcalc), returning every u_k.
 * q_0 = 0; c = e_c; for k = 1..n: q_k = q_{k-1} + c; c <- c - alpha W^T W c;
 * u_k = alpha W q_k.  Written as u_k = u_{k-1} + alpha W c_{k-1} (linearity;
 * reading A6: u_1 = alpha W e_c).  e_c: reading A5 -- for even N the 2x2
 * average of the four central pixels, for odd N the centre pixel.
 * bank: n_k x na x nd.
 * ------------------------------------------------------------------------- */
static void central_impulse(int n, double* c) {
    memset(c, 0, sizeof(double) * (size_t)n * n);
    if (n % 2) {
        c[(size_t)(n / 2) * n + n / 2] = 1.0;
    } else {
        const int m = n / 2;
        c[(size_t)(m - 1) * n + (m - 1)] = 0.25;
        c[(size_t)(m - 1) * n + m] = 0.25;
        c[(size_t)m * n + (m - 1)] = 0.25;
        c[(size_t)m * n + m] = 0.25;
    }
}

int or_filter_bank(int n, int na, int nd, const double* ang, int nk, double alpha, double* bank) {
    if (check_geom(n, na, nd, ang) || nk < 1 || !(alpha > 0.0)) return OR_ERR_INVALID;
    const size_t ns = (size_t)na * nd, ni = (size_t)n * n;
    double* c = (double*)malloc(sizeof(double) * ni);
    double* wtv = (double*)malloc(sizeof(double) * ni);
    double* v = (double*)malloc(sizeof(double) * ns);
    central_impulse(n, c);
    for (int k = 0; k < nk; ++k) {
        fp_rect(n, na, nd, ang, c, n, 0, 0, n, n, v);                 /* v = W c_{k}      */
        double* u = bank + (size_t)k * ns;
        const double* uprev = k ? bank + (size_t)(k - 1) * ns : NULL;
        for (size_t e = 0; e < ns; ++e) u[e] = (uprev ? uprev[e] : 0.0) + alpha * v[e];
        if (k + 1 < nk) {
            bp_rect(n, na, nd, ang, v, wtv, n, 0, 0, n, n);           /* W^T W c          */
            for (size_t e = 0; e < ni; ++e) c[e] -= alpha * wtv[e];  /* c <- c - a W^TW c */
        }
    }
    free(c); free(wtv); free(v);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * C_h: convolve each detector row with that angle's filter row,
 * full linear convolution, zero padded, centre aligned, cropped to N_d:
 *   out(a,d) = sum_j h(a,j) p(a, d - j + d_c),  d_c = (N_d-1)/2  (N_d odd).
 * Direct O(N_d^2) sum: the plain definition.
 * ------------------------------------------------------------------------- */
int or_convolve(int na, int nd, const double* h, const double* p, double* out) {
    if (na < 1 || nd < 1 || nd % 2 == 0) return OR_ERR_INVALID;
    const int dc = (nd - 1) / 2;
#pragma omp parallel for schedule(static)
    for (int a = 0; a < na; ++a) {
        const double* hr = h + (size_t)a * nd;
        const double* pr = p + (size_t)a * nd;
        for (int d = 0; d < nd; ++d) {
            double acc = 0.0;
            for (int j = 0; j < nd; ++j) {
                const int m = d - j + dc;
                if (m >= 0 && m < nd) acc += hr[j] * pr[m];
            }
            out[(size_t)a * nd + d] = acc;
        }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Disc pre-correction (reading A7): D = 1 on pixels whose centre
 * lies in the disc of diameter N centred on the rotation axis; the gray value
 * c minimizes sum_a (P_a - c D_a)^2 over the zero-frequency components
 * P_a = sum_d p(a,d), D_a = sum_d (W D)(a,d); p_c = p - c W D.
 * Outputs: pc [na*nd], c, wd [na*nd] (W D), dimg [N*N] (D).
 * ------------------------------------------------------------------------- */
int or_disc(int n, int na, int nd, const double* ang, const double* p,
            double* pc, double* c_out, double* wd, double* dimg) {
    if (check_geom(n, na, nd, ang)) return OR_ERR_INVALID;
    const double half_n = 0.5 * (n - 1), rad2 = 0.25 * (double)n * n;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double x = j - half_n, y = half_n - i;
            dimg[(size_t)i * n + j] = (x * x + y * y <= rad2) ? 1.0 : 0.0;
        }
    fp_rect(n, na, nd, ang, dimg, n, 0, 0, n, n, wd);
    double num = 0.0, den = 0.0;
    for (int a = 0; a < na; ++a) {
        double pa = 0.0, da = 0.0;
        for (int d = 0; d < nd; ++d) {
            pa += p[(size_t)a * nd + d];
            da += wd[(size_t)a * nd + d];
        }
        num += pa * da;
        den += da * da;
    }
    if (!(den > 0.0)) return OR_ERR_INVALID;
    const double c = num / den;
    for (size_t e = 0; e < (size_t)na * nd; ++e) pc[e] = p[e] - c * wd[e];
    *c_out = c;
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * FGP (Beck & Teboulle 2009, named at P:L661-663; n_FGP = 100 at P:L797-798),
 * anisotropic TV with Neumann boundary on an h x w image (reading A13):
 *   prox: argmin_x 1/2 ||x - b||^2 + lam * TV_aniso(x)
 *   duals p: (h-1) x w, q: h x (w-1); L(p,q)_ij = p_ij + q_ij - p_{i-1,j} - q_{i,j-1}
 *   (out-of-range duals 0); L^T z = (z_ij - z_{i+1,j}, z_ij - z_{i,j+1}).
 *   (r,s) = (p,q) = 0, t = 1; repeat: (p,q)_new = clip_[-1,1]((r,s) + 1/(8 lam) L^T(b - lam L(r,s)));
 *   t' = (1+sqrt(1+4t^2))/2; (r,s) = new + (t-1)/t' (new - old); output b - lam L(p,q).
 * lam = 0 -> identity.  P, Q (nullable) receive the final duals.
 * ------------------------------------------------------------------------- */
static double Lop(const double* p, const double* q, int h, int w, int i, int j) {
    double v = 0.0;
    if (i < h - 1) v += p[(size_t)i * w + j];
    if (j < w - 1) v += q[(size_t)i * (w - 1) + j];
    if (i > 0) v -= p[(size_t)(i - 1) * w + j];
    if (j > 0) v -= q[(size_t)i * (w - 1) + (j - 1)];
    return v;
}

static double clip1(double v) { return v > 1.0 ? 1.0 : (v < -1.0 ? -1.0 : v); }

static void fgp(int h, int w, const double* b, double lam, int nit, double* x, double* P, double* Q) {
    const size_t np = (size_t)(h > 1 ? h - 1 : 0) * w, nq = (size_t)h * (w > 1 ? w - 1 : 0);
    if (lam == 0.0) {
        memcpy(x, b, sizeof(double) * (size_t)h * w);
        if (P) memset(P, 0, sizeof(double) * np);
        if (Q) memset(Q, 0, sizeof(double) * nq);
        return;
    }
    double* p = (double*)calloc(np + 1, sizeof(double));
    double* q = (double*)calloc(nq + 1, sizeof(double));
    double* r = (double*)calloc(np + 1, sizeof(double));
    double* s = (double*)calloc(nq + 1, sizeof(double));
    double* pn = (double*)calloc(np + 1, sizeof(double));
    double* qn = (double*)calloc(nq + 1, sizeof(double));
    double* z = (double*)malloc(sizeof(double) * (size_t)h * w);
    const double g = 1.0 / (8.0 * lam);
    double t = 1.0;
    /* (rows in parallel only for large images: every element is computed by one
     * thread from the previous iterate, so the thread count changes nothing) */
    const int par = (size_t)h * w >= 4096;
    for (int it = 0; it < nit; ++it) {
#pragma omp parallel for schedule(static) if (par)
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) z[(size_t)i * w + j] = b[(size_t)i * w + j] - lam * Lop(r, s, h, w, i, j);
#pragma omp parallel for schedule(static) if (par)
        for (int i = 0; i < h - 1; ++i)
            for (int j = 0; j < w; ++j)
                pn[(size_t)i * w + j] = clip1(r[(size_t)i * w + j] + g * (z[(size_t)i * w + j] - z[(size_t)(i + 1) * w + j]));
#pragma omp parallel for schedule(static) if (par)
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w - 1; ++j)
                qn[(size_t)i * (w - 1) + j] = clip1(s[(size_t)i * (w - 1) + j] + g * (z[(size_t)i * w + j] - z[(size_t)i * w + j + 1]));
        const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
        const double beta = (t - 1.0) / tn;
        for (size_t e = 0; e < np; ++e) { r[e] = pn[e] + beta * (pn[e] - p[e]); p[e] = pn[e]; }
        for (size_t e = 0; e < nq; ++e) { s[e] = qn[e] + beta * (qn[e] - q[e]); q[e] = qn[e]; }
        t = tn;
    }
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) x[(size_t)i * w + j] = b[(size_t)i * w + j] - lam * Lop(p, q, h, w, i, j);
    if (P) memcpy(P, p, sizeof(double) * np);
    if (Q) memcpy(Q, q, sizeof(double) * nq);
    free(p); free(q); free(r); free(s); free(pn); free(qn); free(z);
}

int or_fgp(int h, int w, const double* b, double lam, int nit, double* x, double* P, double* Q) {
    if (h < 1 || w < 1 || lam < 0.0 || nit < 1) return OR_ERR_INVALID;
    fgp(h, w, b, lam, nit, x, P, Q);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * ROI rectangles (P:L246 square local part; P:L706-709 padding, explicit
 * margin per reading A8; clipped to the grid).  rects[8*r]:
 *   core r0, r1, c0, c1, ext r0, r1, c0, c1 (half-open).
 * ------------------------------------------------------------------------- */
int or_roi_rects(int n, int nroi, const int* centres, int radius, int margin, int* rects) {
    if (n < 1 || nroi < 0 || radius < 1 || margin < 0) return OR_ERR_INVALID;
    const int h = radius + margin;
    for (int r = 0; r < nroi; ++r) {
        const int cr = centres[2 * r], cc = centres[2 * r + 1];
        if (cr - radius < 0 || cc - radius < 0 || cr + radius > n || cc + radius > n) return OR_ERR_INVALID;
        int* o = rects + 8 * r;
        o[0] = cr - radius; o[1] = cr + radius; o[2] = cc - radius; o[3] = cc + radius;
        o[4] = cr - h < 0 ? 0 : cr - h;
        o[5] = cr + h > n ? n : cr + h;
        o[6] = cc - h < 0 ? 0 : cc - h;
        o[7] = cc + h > n ? n : cc + h;
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Haar wavelet prior.  B = the orthonormal 2D Haar
 * decomposition with `levels` levels (the paper's "wavelet decomposition
 * operator B", in a Haar basis), on an h x w image with
 * 2^levels dividing h and w, stored in place: level l (stride
 * s = 2^l) maps every 2x2 group of approximation samples (a b; c d) at
 * (i, j), (i, j+s), (i+s, j), (i+s, j+s), i, j multiples of 2s, to
 * ((a+b+c+d)/2, (a-b+c-d)/2, (a+b-c-d)/2, (a-b-c+d)/2).  Its inverse applies
 * the same (self-inverse) 2x2 map from the coarsest level down.
 * P_lambda: symmetric soft threshold of EVERY coefficient (g(x) = ||Bx||_1,
 * P:L764; symmetric per reading A15 of the one-sided P:L409).
 * ------------------------------------------------------------------------- */
static void haar_level(int w, int s, int gi, int gj, double* x) {
    double* a = x + (size_t)gi * w + gj;
    double* b = a + s;
    double* c = a + (size_t)s * w;
    double* d = c + s;
    const double A = *a, B = *b, C = *c, D = *d;
    *a = 0.5 * (A + B + C + D);
    *b = 0.5 * (A - B + C - D);
    *c = 0.5 * (A + B - C - D);
    *d = 0.5 * (A - B - C + D);
}

static void haar_fwd(int h, int w, int levels, double* x) {
    for (int l = 0; l < levels; ++l) {
        const int s = 1 << l;
        for (int i = 0; i < h; i += 2 * s)
            for (int j = 0; j < w; j += 2 * s) haar_level(w, s, i, j, x);
    }
}

static void haar_inv(int h, int w, int levels, double* x) {
    for (int l = levels - 1; l >= 0; --l) {
        const int s = 1 << l;
        for (int i = 0; i < h; i += 2 * s)
            for (int j = 0; j < w; j += 2 * s) haar_level(w, s, i, j, x);
    }
}

/* x = B^{-1} P_lambda(B v)  (eq. sirtista P:L400-401 applied to v = S(.)) */
static void haar_prox(int h, int w, int levels, const double* v, double lam, double* x) {
    const size_t P = (size_t)h * w;
    memcpy(x, v, sizeof(double) * P);
    haar_fwd(h, w, levels, x);
    for (size_t e = 0; e < P; ++e) {
        const double a = fabs(x[e]) - lam;
        x[e] = a > 0.0 ? (x[e] > 0.0 ? a : -a) : 0.0;
    }
    haar_inv(h, w, levels, x);
}

int or_haar(int h, int w, int levels, int inverse, double* x) {
    if (h < 1 || w < 1 || levels < 0 || (h % (1 << levels)) || (w % (1 << levels))) return OR_ERR_INVALID;
    if (inverse) haar_inv(h, w, levels, x); else haar_fwd(h, w, levels, x);
    return OR_OK;
}

int or_haar_prox(int h, int w, int levels, const double* v, double lam, double* x) {
    if (h < 1 || w < 1 || levels < 0 || (h % (1 << levels)) || (w % (1 << levels)) || !(lam >= 0.0))
        return OR_ERR_INVALID;
    haar_prox(h, w, levels, v, lam, x);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Local method for one ROI (eq. localmethod; Alg. 2 P:L637-652 with
 * the box correction d of P:L538-546; Alg. 3 P:L665-688 with the FISTA garbles
 * corrected per reading A12).  The prior acts only on the extended ROI L'
 * (A18).  x_s^k = M W^T b_k + c M D with b_k = C_{u_k} p_c
 * (disc added inside x_s per A7).
 *   mode 0 (box):  S = x_s + y - alpha M W^T W M y;  x = clamp(S,lo,hi);  y = x - x_s
 *   mode 1 (TV):   v = x_s + y - alpha M W^T W M y;  x = FGP(v);  t' = ...;
 *                  r = x + (t-1)/t' (x - x_prev);  y = r - x_s;  x_prev = x
 *                  (momentum = 0 -> r = x)
 *   mode 2 (Haar): as mode 1 with x = B^{-1} P_lam(B v) (NEXT-2; the paper's
 *                  FISTA for the l1 penalties); nfgp = levels
 * Output: x^n on the extended rect (ext_out, h_e x w_e, nullable) and cropped
 * to the core (core_out, 2r x 2r).
 * xs_exact (nullable): nk images N x N replacing x_s^k (pins P9/P10: exact
 * SIRT iterates instead of the filter approximation).
 * ------------------------------------------------------------------------- */
static void local_one(int n, int na, int nd, const double* ang, int nk, double alpha,
                      const double* bconv, double discc, int use_disc, const int* rect,
                      int mode, double lo, double hi, double lam, int nfgp, int momentum,
                      const double* xs_exact, double* ext_out, double* core_out) {
    const int er0 = rect[4], er1 = rect[5], ec0 = rect[6], ec1 = rect[7];
    const int H = er1 - er0, Wd = ec1 - ec0;
    const size_t P = (size_t)H * Wd, ns = (size_t)na * nd;
    const double half_n = 0.5 * (n - 1), rad2 = 0.25 * (double)n * n;
    double* y = (double*)calloc(P, sizeof(double));
    double* xs = (double*)malloc(sizeof(double) * P);
    double* g2 = (double*)calloc(P, sizeof(double));
    double* v = (double*)malloc(sizeof(double) * P);
    double* x = (double*)calloc(P, sizeof(double));
    double* xprev = (double*)calloc(P, sizeof(double));
    double* sino = (double*)malloc(sizeof(double) * ns);
    double t = 1.0;
    for (int k = 0; k < nk; ++k) {
        /* x_s^k = FBP_L(p_c, u_k) + c D  (Alg. 2 line 3; A7) */
        if (xs_exact) {
            const double* xe = xs_exact + (size_t)k * n * n;
            for (int i = 0; i < H; ++i)
                for (int j = 0; j < Wd; ++j) xs[(size_t)i * Wd + j] = xe[(size_t)(er0 + i) * n + ec0 + j];
        } else {
            bp_rect(n, na, nd, ang, bconv + (size_t)k * ns, xs, Wd, er0, ec0, H, Wd);
            if (use_disc)
                for (int i = 0; i < H; ++i)
                    for (int j = 0; j < Wd; ++j) {
                        const double xx = (ec0 + j) - half_n, yy = half_n - (er0 + i);
                        if (xx * xx + yy * yy <= rad2) xs[(size_t)i * Wd + j] += discc;
                    }
        }
        /* y - alpha W_L^T W_L y */
        fp_rect(n, na, nd, ang, y, Wd, er0, ec0, H, Wd, sino);
        bp_rect(n, na, nd, ang, sino, g2, Wd, er0, ec0, H, Wd);
        for (size_t e = 0; e < P; ++e) v[e] = xs[e] + y[e] - alpha * g2[e];
        if (mode == 0) {
            /* d^k = clamp(S) - S  =>  y^k = clamp(S) - x_s^k */
            for (size_t e = 0; e < P; ++e) {
                double s = v[e];
                x[e] = s < lo ? lo : (s > hi ? hi : s);
                y[e] = x[e] - xs[e];
            }
        } else {
            if (mode == 2) haar_prox(H, Wd, nfgp, v, lam, x);      /* Haar prior: nfgp = levels (NEXT-2) */
            else fgp(H, Wd, v, lam, nfgp, x, NULL, NULL);          /* Alg. 3 line 6 */
            const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)); /* A12 */
            const double beta = momentum ? (t - 1.0) / tn : 0.0;
            for (size_t e = 0; e < P; ++e) {
                const double r = x[e] + beta * (x[e] - xprev[e]);
                y[e] = r - xs[e];
                xprev[e] = x[e];
            }
            t = tn;
        }
    }
    if (ext_out) memcpy(ext_out, x, sizeof(double) * P);
    if (core_out) {
        const int side = rect[1] - rect[0];
        for (int i = 0; i < side; ++i)
            for (int j = 0; j < side; ++j)
                core_out[(size_t)i * side + j] = x[(size_t)(rect[0] + i - er0) * Wd + (rect[2] + j - ec0)];
    }
    free(y); free(xs); free(g2); free(v); free(x); free(xprev); free(sino);
}

/* Local solves for nroi ROIs.  bconv: nk x na x nd conv cache (b_k, k = 1..nk).
 * cores: nroi x (2r)^2.  ext (nullable): nroi x (2h)^2, each ROI's valid
 * extended rect stored top-left aligned with row stride 2h, zeros elsewhere. */
int or_local_solve(int n, int na, int nd, const double* ang, int nk, double alpha,
                   const double* bconv, double discc, int use_disc,
                   int nroi, const int* centres, int radius, int margin,
                   int mode, double lo, double hi, double lam, int nfgp, int momentum,
                   const double* xs_exact, double* cores, double* ext) {
    if (check_geom(n, na, nd, ang) || nk < 1 || !(alpha > 0.0)) return OR_ERR_INVALID;
    if (mode == 0 && lo > hi) return OR_ERR_INVALID;
    if (mode == 1 && (lam < 0.0 || nfgp < 1)) return OR_ERR_INVALID;
    if (mode == 2 && (lam < 0.0 || nfgp < 0)) return OR_ERR_INVALID;
    int* rects = (int*)malloc(sizeof(int) * 8 * (nroi > 0 ? nroi : 1));
    if (or_roi_rects(n, nroi, centres, radius, margin, rects)) { free(rects); return OR_ERR_INVALID; }
    const int side = 2 * radius, eside = 2 * (radius + margin);
    if (mode == 2)
        for (int r = 0; r < nroi; ++r) {
            const int* rc = rects + 8 * r;
            if ((rc[5] - rc[4]) % (1 << nfgp) || (rc[7] - rc[6]) % (1 << nfgp)) { free(rects); return OR_ERR_INVALID; }
        }
    for (int r = 0; r < nroi; ++r) {
        const int* rc = rects + 8 * r;
        const int H = rc[5] - rc[4], Wd = rc[7] - rc[6];
        double* tmp = ext ? (double*)malloc(sizeof(double) * (size_t)H * Wd) : NULL;
        local_one(n, na, nd, ang, nk, alpha, bconv, discc, use_disc, rc, mode, lo, hi, lam, nfgp,
                  momentum, xs_exact, tmp, cores + (size_t)r * side * side);
        if (ext) {
            double* e = ext + (size_t)r * eside * eside;
            memset(e, 0, sizeof(double) * (size_t)eside * eside);
            for (int i = 0; i < H; ++i)
                for (int j = 0; j < Wd; ++j) e[(size_t)i * eside + j] = tmp[(size_t)i * Wd + j];
            free(tmp);
        }
    }
    free(rects);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Global solvers the method approximates (reading a10):
 *   box-SIRT  x^{k+1} = clamp(x^k + alpha W^T (p - W x^k))   (eq. sirtbox P:L382-396,
 *             eq. sirtit, x^0 = 0 per A17)
 *   FISTA-TV  x^k = FGP(S(r^{k-1})), r^k = x^k + (t_{k-1}-1)/t_k (x^k - x^{k-1})
 *             (A12, A14)
 * iterates (nullable): all x^k, k = 1..nk (nk x N x N), used by pins P9/P10.
 * ------------------------------------------------------------------------- */
static void sirt_step(int n, int na, int nd, const double* ang, double alpha,
                      const double* p, const double* x, double* out, double* sino, double* bp) {
    const size_t ns = (size_t)na * nd, ni = (size_t)n * n;
    fp_rect(n, na, nd, ang, x, n, 0, 0, n, n, sino);
    for (size_t e = 0; e < ns; ++e) sino[e] = p[e] - sino[e];
    bp_rect(n, na, nd, ang, sino, bp, n, 0, 0, n, n);
    for (size_t e = 0; e < ni; ++e) out[e] = x[e] + alpha * bp[e];
}

int or_global_box(int n, int na, int nd, const double* ang, const double* p, int nk, double alpha,
                  double lo, double hi, double* x, double* iterates) {
    if (check_geom(n, na, nd, ang) || nk < 1 || lo > hi) return OR_ERR_INVALID;
    const size_t ns = (size_t)na * nd, ni = (size_t)n * n;
    double* sino = (double*)malloc(sizeof(double) * ns);
    double* bp = (double*)malloc(sizeof(double) * ni);
    double* s = (double*)malloc(sizeof(double) * ni);
    memset(x, 0, sizeof(double) * ni);
    for (int k = 0; k < nk; ++k) {
        sirt_step(n, na, nd, ang, alpha, p, x, s, sino, bp);
        for (size_t e = 0; e < ni; ++e) x[e] = s[e] < lo ? lo : (s[e] > hi ? hi : s[e]);
        if (iterates) memcpy(iterates + (size_t)k * ni, x, sizeof(double) * ni);
    }
    free(sino); free(bp); free(s);
    return OR_OK;
}

int or_global_tv(int n, int na, int nd, const double* ang, const double* p, int nk, double alpha,
                 double lam, int nfgp, int momentum, double* x) {
    if (check_geom(n, na, nd, ang) || nk < 1 || lam < 0.0 || nfgp < 1) return OR_ERR_INVALID;
    const size_t ns = (size_t)na * nd, ni = (size_t)n * n;
    double* sino = (double*)malloc(sizeof(double) * ns);
    double* bp = (double*)malloc(sizeof(double) * ni);
    double* s = (double*)malloc(sizeof(double) * ni);
    double* r = (double*)calloc(ni, sizeof(double));
    double* xprev = (double*)calloc(ni, sizeof(double));
    double t = 1.0;
    for (int k = 0; k < nk; ++k) {
        sirt_step(n, na, nd, ang, alpha, p, r, s, sino, bp);
        fgp(n, n, s, lam, nfgp, x, NULL, NULL);
        const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
        const double beta = momentum ? (t - 1.0) / tn : 0.0;
        for (size_t e = 0; e < ni; ++e) {
            r[e] = x[e] + beta * (x[e] - xprev[e]);
            xprev[e] = x[e];
        }
        t = tn;
    }
    free(sino); free(bp); free(s); free(r); free(xprev);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Exterior subtraction (the prior art of P:L140-146,
 * "subtracting simulated projections of a global reconstruction outside the
 * region of interest from the acquired projections ... used in an algebraic
 * reconstruction of the region of interest").  Given a global reconstruction
 * xg (N x N), for every ROI with extended rect L':
 *     p~ = p - W M_F xg          (M_F = 1 - M_{L'}: the exterior)
 *     x  <- clamp(x + alpha M_{L'} W^T (p~ - W M_{L'} x), lo, hi),  x^0 = 0, nk times
 * (box-SIRT, eq. sirtbox, on L'); cores cropped as or_local_solve.
 * ------------------------------------------------------------------------- */
int or_exterior_solve(int n, int na, int nd, const double* ang, const double* p, const double* xg, int nroi,
                      const int* centres, int radius, int margin, int nk, double alpha, double lo, double hi,
                      double* cores) {
    if (check_geom(n, na, nd, ang) || nk < 1 || lo > hi || !(alpha > 0.0)) return OR_ERR_INVALID;
    int* rects = (int*)malloc(sizeof(int) * 8 * (nroi > 0 ? nroi : 1));
    if (or_roi_rects(n, nroi, centres, radius, margin, rects)) { free(rects); return OR_ERR_INVALID; }
    const size_t ns = (size_t)na * nd, ni = (size_t)n * n;
    double* ext = (double*)malloc(sizeof(double) * ni);
    double* pt = (double*)malloc(sizeof(double) * ns);
    double* sino = (double*)malloc(sizeof(double) * ns);
    const int side = 2 * radius;
    for (int r = 0; r < nroi; ++r) {
        const int* rc = rects + 8 * r;
        const int er0 = rc[4], er1 = rc[5], ec0 = rc[6], ec1 = rc[7];
        const int H = er1 - er0, Wd = ec1 - ec0;
        const size_t P = (size_t)H * Wd;
        /* M_F xg: the global reconstruction with the extended ROI zeroed */
        memcpy(ext, xg, sizeof(double) * ni);
        for (int i = er0; i < er1; ++i)
            for (int j = ec0; j < ec1; ++j) ext[(size_t)i * n + j] = 0.0;
        fp_rect(n, na, nd, ang, ext, n, 0, 0, n, n, sino);
        for (size_t e = 0; e < ns; ++e) pt[e] = p[e] - sino[e];
        double* x = (double*)calloc(P, sizeof(double));
        double* g = (double*)malloc(sizeof(double) * P);
        for (int k = 0; k < nk; ++k) {
            fp_rect(n, na, nd, ang, x, Wd, er0, ec0, H, Wd, sino);
            for (size_t e = 0; e < ns; ++e) sino[e] = pt[e] - sino[e];
            bp_rect(n, na, nd, ang, sino, g, Wd, er0, ec0, H, Wd);
            for (size_t e = 0; e < P; ++e) {
                const double s = x[e] + alpha * g[e];
                x[e] = s < lo ? lo : (s > hi ? hi : s);
            }
        }
        for (int i = 0; i < side; ++i)
            for (int j = 0; j < side; ++j)
                cores[(size_t)r * side * side + (size_t)i * side + j] = x[(size_t)(rc[0] + i - er0) * Wd + (rc[2] + j - ec0)];
        free(x); free(g);
    }
    free(rects); free(ext); free(pt); free(sino);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Chambolle-Pock primal-dual TV solver with diagonal preconditioning (SURVEY
 * §8(f) NEXT-4(iii): the north star's literal "TV-regularized primal-dual
 * solver ... row and column normalisation"; Chambolle & Pock 2011 and Pock &
 * Chambolle 2011, alpha = 1; the paper names primal-dual methods at P:L351-353
 * and sets them aside because they are not "SIRT step + correction" methods,
 * P:L371-381, so this is a GLOBAL solver only).  It minimises the same
 * objective as the FISTA-TV reading A14:
 *     F(x) = 1/2 ||W x - p||^2 + mu ||grad x||_1,   mu = lam / alpha,
 * anisotropic forward differences with Neumann boundary (A13), no constraint.
 * K = [W; grad]; Sigma = 1 / row sums of |K| (rays: sum_j W_ij = W 1; TV
 * duals: 1/2), T = 1 / column sums (W^T 1 + number of difference terms that
 * touch the pixel).  From x = xbar = 0, yd = 0, (yp, yq) = 0:
 *     yd <- (yd + sd (W xbar - p)) / (1 + sd)           prox of (1/2||.-p||^2)*
 *     (yp, yq) <- clip_[-mu, mu]((yp, yq) + 1/2 grad xbar)
 *     x' <- x - T (W^T yd + grad^T (yp, yq));  xbar <- 2 x' - x;  x <- x'
 * grad^T (p, q)_ij = p_ij + q_ij - p_{i-1,j} - q_{i,j-1} (the L of the FGP).
 * ------------------------------------------------------------------------- */
int or_global_cp(int n, int na, int nd, const double* ang, const double* p, int nk, double mu, double* x) {
    if (check_geom(n, na, nd, ang) || nk < 1 || !(mu >= 0.0)) return OR_ERR_INVALID;
    const size_t ns = (size_t)na * nd, ni = (size_t)n * n;
    double* ones = (double*)malloc(sizeof(double) * ni);
    double* sd = (double*)malloc(sizeof(double) * ns);
    double* tau = (double*)malloc(sizeof(double) * ni);
    double* yd = (double*)calloc(ns, sizeof(double));
    double* yp = (double*)calloc(ni, sizeof(double));
    double* yq = (double*)calloc(ni, sizeof(double));
    double* xb = (double*)calloc(ni, sizeof(double));
    double* sino = (double*)malloc(sizeof(double) * ns);
    double* g = (double*)malloc(sizeof(double) * ni);
    for (size_t e = 0; e < ni; ++e) ones[e] = 1.0;
    fp_rect(n, na, nd, ang, ones, n, 0, 0, n, n, sino);                 /* row sums W 1 */
    for (size_t e = 0; e < ns; ++e) sd[e] = sino[e] > 0.0 ? 1.0 / sino[e] : 0.0;
    for (size_t e = 0; e < ns; ++e) sino[e] = 1.0;
    bp_rect(n, na, nd, ang, sino, tau, n, 0, 0, n, n);                  /* column sums W^T 1 */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int terms = (i < n - 1) + (i > 0) + (j < n - 1) + (j > 0);
            tau[(size_t)i * n + j] = 1.0 / (tau[(size_t)i * n + j] + terms);
        }
    memset(x, 0, sizeof(double) * ni);
    for (int k = 0; k < nk; ++k) {
        fp_rect(n, na, nd, ang, xb, n, 0, 0, n, n, sino);
        for (size_t e = 0; e < ns; ++e) yd[e] = (yd[e] + sd[e] * (sino[e] - p[e])) / (1.0 + sd[e]);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const size_t o = (size_t)i * n + j;
                const double dx = i < n - 1 ? xb[o + n] - xb[o] : 0.0;   /* p: vertical forward difference */
                const double dy = j < n - 1 ? xb[o + 1] - xb[o] : 0.0;   /* q: horizontal */
                double a = yp[o] + 0.5 * dx, b = yq[o] + 0.5 * dy;
                yp[o] = i < n - 1 ? (a > mu ? mu : (a < -mu ? -mu : a)) : 0.0;
                yq[o] = j < n - 1 ? (b > mu ? mu : (b < -mu ? -mu : b)) : 0.0;
            }
        bp_rect(n, na, nd, ang, yd, g, n, 0, 0, n, n);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const size_t o = (size_t)i * n + j;
                /* grad^T: the forward-difference transpose (-div) */
                const double gt = -(yp[o] + yq[o]) + (i > 0 ? yp[o - n] : 0.0) + (j > 0 ? yq[o - 1] : 0.0);
                const double xn = x[o] - tau[o] * (g[o] + gt);
                xb[o] = 2.0 * xn - x[o];
                x[o] = xn;
            }
    }
    free(ones); free(sd); free(tau); free(yd); free(yp); free(yq); free(xb); free(sino); free(g);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Combine (P:L1122-1127 tiling by placement; reading A19 for overlaps):
 * img(i,j) = mean over the ROIs whose core contains (i,j), summed in
 * ascending ROI index; pixels covered by no core are 0.
 * ------------------------------------------------------------------------- */
int or_stitch(int n, int nroi, const int* centres, int radius, const double* cores, double* img) {
    if (n < 1 || radius < 1) return OR_ERR_INVALID;
    const int side = 2 * radius;
    double* cnt = (double*)calloc((size_t)n * n, sizeof(double));
    memset(img, 0, sizeof(double) * (size_t)n * n);
    for (int r = 0; r < nroi; ++r) {
        const int r0 = centres[2 * r] - radius, c0 = centres[2 * r + 1] - radius;
        if (r0 < 0 || c0 < 0 || r0 + side > n || c0 + side > n) { free(cnt); return OR_ERR_INVALID; }
        for (int i = 0; i < side; ++i)
            for (int j = 0; j < side; ++j) {
                img[(size_t)(r0 + i) * n + c0 + j] += cores[(size_t)r * side * side + (size_t)i * side + j];
                cnt[(size_t)(r0 + i) * n + c0 + j] += 1.0;
            }
    }
    for (size_t e = 0; e < (size_t)n * n; ++e)
        if (cnt[e] > 0.0) img[e] /= cnt[e];
    free(cnt);
    return OR_OK;
}
