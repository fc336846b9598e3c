/*
 * oracle.c -- CPU oracle for hybrid-dealiased convolution (arXiv 2306.10016).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (libhdconv.so, paper_2306_10016_b200/) never links,
 * imports or calls it, and it shares no code, header, table or helper with
 * the CUDA path.
 *
 * What it computes: the plain definition the method reaches exactly.
 *   Hybrid dealiasing removes the aliases (the s != 0 terms of PAPER.md:547,
 *   "The terms indexed by s != 0 are aliases") whenever the
 *   padded size M >= L_f + L_g - 1, so the method's output is
 *   the linear convolution of Eq. (4), PAPER.md:537-541:
 *        (f*g)_k = sum_p f_p g_{k-p},
 *   extended per axis to N dimensions ("the same parameters for
 *   each dimension") and summed over pairs for multi-convolution
 *   (reading R9: h = sum_k f_k * g_k, BASELINE.json configs[4]).
 *   The full output has extent L_f,i + L_g,i - 1 on every axis
 *   (reading R3).
 *
 * Arithmetic: complex double (interleaved re, im), one complex MAC per
 * term, summed innermost axis first, then row partials, then plane partials
 * (blocked only to bound round-off; no reordering beyond that).
 * complex64 inputs are upcast exactly by the Python wrapper.
 *
 * Also here: the naive DFT of PAPER.md:501-503 (Eq. 1, positive exponent,
 * unnormalised) used to pin the CUDA residue transforms (block r of the
 * hybrid forward transform = DFT_{qm}(x zero-padded)[q*l + r]),
 * and Horner evaluation of the generating polynomial
 * P_a(z) = sum_o a[o] prod_i z_i^{o_i} (closed-form pin P_h = P_f * P_g).
 *
 * Parallelism: OpenMP over output samples; every sample is independent.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MAXDIM 3

typedef struct { double re, im; } cplx;

static inline void cmac(cplx* acc, cplx a, cplx b) {
  acc->re += a.re * b.re - a.im * b.im;
  acc->im += a.re * b.im + a.im * b.re;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Pad the shape description to 3 axes: extents (1,...,1,L...). */
static void pad3(int ndim, const int64_t* L, int64_t out[3]) {
  for (int i = 0; i < 3; ++i) out[i] = 1;
  for (int i = 0; i < ndim; ++i) out[3 - ndim + i] = L[i];
}

/* One output sample o (3 padded indices) of sum_k f_k * g_k (Eq. 4 per axis). */
static cplx conv_at(int npairs, const int64_t Af[3], const cplx* const* f,
                    const int64_t Ag[3], const cplx* const* g, const int64_t o[3]) {
  cplx total = {0.0, 0.0};
  int64_t lo[3], hi[3];
  for (int i = 0; i < 3; ++i) {
    /* valid a_i: 0 <= a_i < Af_i and 0 <= o_i - a_i < Ag_i */
    lo[i] = o[i] - (Ag[i] - 1); if (lo[i] < 0) lo[i] = 0;
    hi[i] = o[i];               if (hi[i] > Af[i] - 1) hi[i] = Af[i] - 1;
    if (lo[i] > hi[i]) return total;
  }
  for (int k = 0; k < npairs; ++k) {          /* pairs in fixed order k = 0..N-1 */
    cplx plane = {0.0, 0.0};
    for (int64_t a0 = lo[0]; a0 <= hi[0]; ++a0) {
      cplx row = {0.0, 0.0};
      for (int64_t a1 = lo[1]; a1 <= hi[1]; ++a1) {
        cplx acc = {0.0, 0.0};
        const cplx* fr = f[k] + (a0 * Af[1] + a1) * Af[2];
        const cplx* gr = g[k] + ((o[0] - a0) * Ag[1] + (o[1] - a1)) * Ag[2];
        for (int64_t a2 = lo[2]; a2 <= hi[2]; ++a2) cmac(&acc, fr[a2], gr[o[2] - a2]);
        row.re += acc.re; row.im += acc.im;
      }
      plane.re += row.re; plane.im += row.im;
    }
    total.re += plane.re; total.im += plane.im;
  }
  return total;
}

/* h = sum_{k<npairs} f_k * g_k, full extent Lf_i + Lg_i - 1 on each axis.
 * f[k], g[k]: interleaved complex double arrays, row-major, last axis fastest.
 * Returns 0 on success, -1 on bad arguments. */
int oracle_multiconv(int ndim, int npairs, const int64_t* Lf, const double* const* f,
                     const int64_t* Lg, const double* const* g, double* h) {
  if (ndim < 1 || ndim > ORACLE_MAXDIM || npairs < 1) return -1;
  for (int i = 0; i < ndim; ++i) if (Lf[i] < 1 || Lg[i] < 1) return -1;
  int64_t Af[3], Ag[3], Ao[3];
  pad3(ndim, Lf, Af); pad3(ndim, Lg, Ag);
  for (int i = 0; i < 3; ++i) Ao[i] = Af[i] + Ag[i] - 1;
  const int64_t nout = Ao[0] * Ao[1] * Ao[2];
  const cplx* const* fc = (const cplx* const*)f;
  const cplx* const* gc = (const cplx* const*)g;
  cplx* hc = (cplx*)h;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t idx = 0; idx < nout; ++idx) {
    int64_t o[3];
    o[2] = idx % Ao[2];
    o[1] = (idx / Ao[2]) % Ao[1];
    o[0] = idx / (Ao[2] * Ao[1]);
    hc[idx] = conv_at(npairs, Af, fc, Ag, gc, o);
  }
  return 0;
}

int oracle_conv(int ndim, const int64_t* Lf, const double* f, const int64_t* Lg,
                const double* g, double* h) {
  const double* fs[1] = {f};
  const double* gs[1] = {g};
  return oracle_multiconv(ndim, 1, Lf, fs, Lg, gs, h);
}

/* The same formula at nsamp given output indices idx[s*ndim + i]. */
int oracle_multiconv_sampled(int ndim, int npairs, const int64_t* Lf, const double* const* f,
                             const int64_t* Lg, const double* const* g, int64_t nsamp,
                             const int64_t* idx, double* out) {
  if (ndim < 1 || ndim > ORACLE_MAXDIM || npairs < 1) return -1;
  int64_t Af[3], Ag[3];
  pad3(ndim, Lf, Af); pad3(ndim, Lg, Ag);
  for (int64_t s = 0; s < nsamp; ++s)
    for (int i = 0; i < ndim; ++i) {
      int64_t v = idx[s * ndim + i];
      if (v < 0 || v >= Lf[i] + Lg[i] - 1) return -1;
    }
  const cplx* const* fc = (const cplx* const*)f;
  const cplx* const* gc = (const cplx* const*)g;
  cplx* oc = (cplx*)out;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < nsamp; ++s) {
    int64_t o[3] = {0, 0, 0};
    for (int i = 0; i < ndim; ++i) o[3 - ndim + i] = idx[s * ndim + i];
    oc[s] = conv_at(npairs, Af, fc, Ag, gc, o);
  }
  return 0;
}

/* Naive DFT, PAPER.md:501-503 (Eq. 1): X_k = sum_{j<L} zeta_M^{sign*k*j} x_j,
 * zeta_M = exp(2 pi i / M), for k < M; x is zero beyond L (L <= M).
 * Exponent k*j is reduced mod M in 64-bit integers before the angle is formed.
 * sign = +1 is the paper's forward transform, -1 its (unnormalised) backward. */
int oracle_dft(int64_t M, int64_t L, const double* x, int sign, double* X) {
  if (M < 1 || L < 0 || L > M || (sign != 1 && sign != -1)) return -1;
  const cplx* xc = (const cplx*)x;
  cplx* Xc = (cplx*)X;
  const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < M; ++k) {
    cplx acc = {0.0, 0.0};
    for (int64_t j = 0; j < L; ++j) {
      int64_t e = (k * j) % M;
      double ang = two_pi * (double)e / (double)M;
      cplx w = {cos(ang), sign * sin(ang)};
      cmac(&acc, xc[j], w);
    }
    Xc[k] = acc;
  }
  return 0;
}

/* P_a(z) = sum_o a[o] prod_i z_i^{o_i} by nested Horner, at npts points
 * z[p*ndim + i] (complex).  Used for the polynomial identity P_h = P_f * P_g.
 * Accumulated in long double (x86-64: 64-bit mantissa) so that the Horner
 * rounding, (sum_i deg_i) * oracle_poly_eps() * ||a||_1 for |z_i| = 1, stays far
 * below the parity tolerances even for 10^7-sample outputs; the result is
 * rounded to double once. */
typedef struct { long double re, im; } lcplx;

double oracle_poly_eps(void) { return (double)LDBL_EPSILON; }

int oracle_poly_eval(int ndim, const int64_t* L, const double* a, int64_t npts,
                     const double* z, double* out) {
  if (ndim < 1 || ndim > ORACLE_MAXDIM) return -1;
  int64_t A[3];
  pad3(ndim, L, A);
  const cplx* ac = (const cplx*)a;
  const cplx* zc = (const cplx*)z;
  cplx* oc = (cplx*)out;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t p = 0; p < npts; ++p) {
    lcplx zz[3] = {{1, 0}, {1, 0}, {1, 0}};
    for (int i = 0; i < ndim; ++i) {
      zz[3 - ndim + i].re = zc[p * ndim + i].re;
      zz[3 - ndim + i].im = zc[p * ndim + i].im;
    }
    lcplx s0 = {0, 0};
    for (int64_t a0 = A[0] - 1; a0 >= 0; --a0) {
      lcplx s1 = {0, 0};
      for (int64_t a1 = A[1] - 1; a1 >= 0; --a1) {
        lcplx s2 = {0, 0};
        const cplx* row = ac + (a0 * A[1] + a1) * A[2];
        for (int64_t a2 = A[2] - 1; a2 >= 0; --a2) {
          lcplx t = {s2.re * zz[2].re - s2.im * zz[2].im, s2.re * zz[2].im + s2.im * zz[2].re};
          s2.re = t.re + row[a2].re; s2.im = t.im + row[a2].im;
        }
        lcplx t = {s1.re * zz[1].re - s1.im * zz[1].im, s1.re * zz[1].im + s1.im * zz[1].re};
        s1.re = t.re + s2.re; s1.im = t.im + s2.im;
      }
      lcplx t = {s0.re * zz[0].re - s0.im * zz[0].im, s0.re * zz[0].im + s0.im * zz[0].re};
      s0.re = t.re + s1.re; s0.im = t.im + s1.im;
    }
    oc[p].re = (double)s0.re;
    oc[p].im = (double)s0.im;
  }
  return 0;
}
