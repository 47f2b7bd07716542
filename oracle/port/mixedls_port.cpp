// oracle/port/mixedls_port.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/orc_api.h).
//
// A CPU restatement of the reference's classical-IR hot path, written as the
// checker for the B200 product.  Real instantiations follow the reference's
// floating-point operation order step by step, so with -ffp-contract=off they
// are bitwise identical to oracle/_ref (tests/test_oracle.py pins that); the
// complex instantiations generalize every transpose to a conjugate transpose
// and the reflectors to xLARFG's complex form (real beta, complex tau), which
// the reference does not have -- they are pinned against a dense
// complex KKT solve and scipy instead.
//
// Algorithm sources (all paths relative to /root/reference/proj/include/mixedls):
//   reflector generation            householder.hpp:30-53
//   rank-1 reflector applications   householder.hpp:56-95
//   factor applies (Q x, Q^T x, ..)  householder.hpp:114-152
//   unblocked QR / RQ               householder.hpp:173-190, :202-222
//   GRQ / GQR                       factor.hpp:34-75, promotion :79-112
//   gemv / gemv_sub / trsv_sub      matrix.hpp:132-154, :215-267
//   extended (double-double) dot    precision.hpp:131-175
//   LSE: direct, cascade, solve_v, residuals, stop test, driver   lse.hpp:48-429
//   GLS: direct, init_z, cascade, residuals, stop test, driver    gls.hpp:47-387
//   refinement plumbing (scales, divergence)                       refine.hpp:79-119
//   seeded generator                 generate.hpp:46-106, random.hpp:16-30
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../orc_api.h"

namespace port {

using i64 = int64_t;
using cd = std::complex<double>;
using cf = std::complex<float>;

// ---- error types mirroring inc/errors.hpp ----------------------------------
struct dim_err : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct bad_input : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct zero_pivot : std::runtime_error {
    explicit zero_pivot(i64 i) : std::runtime_error("zero pivot"), idx(i) {}
    i64 idx;
};

// ---- scalar helpers (identity on reals) ------------------------------------
template <class S> struct traits {
    using real = S;
    using wide = double;
    using low = float;
    static constexpr bool cplx = false;
};
template <class R> struct traits<std::complex<R>> {
    using real = R;
    using wide = cd;
    using low = cf;
    static constexpr bool cplx = true;
};

inline float cj(float x) { return x; }
inline double cj(double x) { return x; }
inline cf cj(cf x) { return std::conj(x); }
inline cd cj(cd x) { return std::conj(x); }
inline double sq(float x) { return double(x) * double(x); }
inline double sq(double x) { return x * x; }
inline double sq(cf x) { return double(x.real()) * double(x.real()) + double(x.imag()) * double(x.imag()); }
inline double sq(cd x) { return x.real() * x.real() + x.imag() * x.imag(); }
inline double mag(double x) { return std::abs(x); }
inline double mag(float x) { return std::abs(double(x)); }
inline double mag(cd x) { return std::abs(x); }
inline double mag(cf x) { return std::abs(cd(x)); }
inline bool finite(double x) { return std::isfinite(x); }
inline bool finite(float x) { return std::isfinite(x); }
inline bool finite(cd x) { return std::isfinite(x.real()) && std::isfinite(x.imag()); }
inline bool finite(cf x) { return std::isfinite(x.real()) && std::isfinite(x.imag()); }

template <class To, class From> To cast(From x) { return static_cast<To>(x); }
template <> inline cf cast<cf, cd>(cd x) { return cf(float(x.real()), float(x.imag())); }
template <> inline cd cast<cd, cf>(cf x) { return cd(double(x.real()), double(x.imag())); }

template <class S> using vec = std::vector<S>;

template <class S> struct mat {
    i64 r = 0, c = 0;
    vec<S> a;
    mat() = default;
    mat(i64 rows, i64 cols) : r(rows), c(cols), a(size_t(rows * cols), S(0)) {}
    S& operator()(i64 i, i64 j) { return a[size_t(j * r + i)]; }
    const S& operator()(i64 i, i64 j) const { return a[size_t(j * r + i)]; }
    S* col(i64 j) { return a.data() + j * r; }
    const S* col(i64 j) const { return a.data() + j * r; }
};

template <class To, class From> vec<To> cast_v(const vec<From>& v) {
    vec<To> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = cast<To>(v[i]);
    return o;
}
template <class To, class From> mat<To> cast_m(const mat<From>& M) {
    mat<To> o(M.r, M.c);
    for (size_t k = 0; k < M.a.size(); ++k) o.a[k] = cast<To>(M.a[k]);
    return o;
}

template <class S> double nrm2(const vec<S>& v) {
    double s = 0.0;
    for (const S& x : v) s += sq(x);
    return std::sqrt(s);
}
template <class S> double nrmF(const mat<S>& M) { return nrm2(M.a); }
// max |x|, skipping NaN like std::max(m, |x|) does
template <class S> double amax(const vec<S>& v) {
    double m = 0.0;
    for (const S& x : v) {
        const double t = mag(x);
        m = (m < t) ? t : m;
    }
    return m;
}
template <class S> bool all_fin(const vec<S>& v) {
    for (const S& x : v)
        if (!finite(x)) return false;
    return true;
}
inline double one_if_zero(double s) { return s == 0.0 ? 1.0 : s; }

// ---- Householder reflectors ------------------------------------------------
// H = I - tau v v^H on [off, off + v.size()), explicit unit entry.
template <class S> struct hh {
    i64 off = 0;
    vec<S> v;
    S tau = S(0);
};

// xLARFG: H^H (alpha; x) = (beta; 0), beta real.  Norm in binary64.
template <class S> S make_hh(S alpha, const S* x, i64 len, bool unit_last, hh<S>& out) {
    double xn = 0.0;
    for (i64 i = 0; i < len; ++i) xn += sq(x[i]);
    xn = std::sqrt(xn);
    out.v.assign(size_t(len + 1), S(0));
    const i64 unit = unit_last ? len : 0;
    if constexpr (!traits<S>::cplx) {
        if (xn == 0.0) {
            out.tau = S(0);
            out.v[size_t(unit)] = S(1);
            return alpha;
        }
        const double a = double(alpha);
        const double beta = -std::copysign(std::hypot(a, xn), a);
        out.tau = static_cast<S>((beta - a) / beta);
        const S inv = static_cast<S>(1.0 / (a - beta));
        for (i64 i = 0; i < len; ++i) out.v[size_t(unit_last ? i : i + 1)] = x[i] * inv;
        out.v[size_t(unit)] = S(1);
        return static_cast<S>(beta);
    } else {
        const double ar = double(alpha.real()), ai = double(alpha.imag());
        if (xn == 0.0 && ai == 0.0) {
            out.tau = S(0);
            out.v[size_t(unit)] = S(1);
            return alpha;
        }
        const double beta = -std::copysign(std::hypot(std::hypot(ar, ai), xn), ar);
        out.tau = cast<S>(cd((beta - ar) / beta, -ai / beta));
        const S inv = cast<S>(cd(1.0, 0.0) / (cd(ar, ai) - cd(beta, 0.0)));
        for (i64 i = 0; i < len; ++i) out.v[size_t(unit_last ? i : i + 1)] = x[i] * inv;
        out.v[size_t(unit)] = S(1);
        return S(typename traits<S>::real(beta));
    }
}

// x := (I - t v v^H) x on the window
template <class S> void hh_vec(const hh<S>& h, S t, vec<S>& x) {
    if (h.tau == S(0)) return;
    S s = S(0);
    for (size_t i = 0; i < h.v.size(); ++i) s += cj(h.v[i]) * x[size_t(h.off) + i];
    s *= t;
    for (size_t i = 0; i < h.v.size(); ++i) x[size_t(h.off) + i] -= s * h.v[i];
}
// A(0:rend, :) := A (I - t v v^H)
template <class S> void hh_right(const hh<S>& h, S t, mat<S>& A, i64 rend) {
    if (h.tau == S(0)) return;
    const i64 len = i64(h.v.size());
    vec<S> w(size_t(rend), S(0));
    for (i64 j = 0; j < len; ++j) {
        const S vj = h.v[size_t(j)];
        const S* aj = A.col(h.off + j);
        for (i64 i = 0; i < rend; ++i) w[size_t(i)] += vj * aj[i];
    }
    for (i64 j = 0; j < len; ++j) {
        const S tvj = t * cj(h.v[size_t(j)]);
        S* aj = A.col(h.off + j);
        for (i64 i = 0; i < rend; ++i) aj[i] -= tvj * w[size_t(i)];
    }
}
// A(:, c0:) := (I - t v v^H) A
template <class S> void hh_left(const hh<S>& h, S t, mat<S>& A, i64 c0) {
    if (h.tau == S(0)) return;
    for (i64 j = c0; j < A.c; ++j) {
        S* aj = A.col(j);
        S s = S(0);
        for (size_t i = 0; i < h.v.size(); ++i) s += cj(h.v[i]) * aj[size_t(h.off) + i];
        s *= t;
        for (size_t i = 0; i < h.v.size(); ++i) aj[size_t(h.off) + i] -= s * h.v[i];
    }
}

// Unitary factor Q = G_0 G_1 ... G_{k-1}, G_j = I - tau_j v_j v_j^H.
template <class S> struct ufac {
    i64 dim = 0;
    vec<hh<S>> g;
    // x := Q x  or  Q^H x
    void apply(vec<S>& x, bool herm) const {
        const i64 k = i64(g.size());
        if (!herm)
            for (i64 j = k; j-- > 0;) hh_vec(g[size_t(j)], g[size_t(j)].tau, x);
        else
            for (i64 j = 0; j < k; ++j) hh_vec(g[size_t(j)], cj(g[size_t(j)].tau), x);
    }
    vec<S> times(const vec<S>& x, bool herm) const {
        if (i64(x.size()) != dim) throw dim_err("factor apply: length mismatch");
        vec<S> y = x;
        apply(y, herm);
        return y;
    }
    // A := Q A  or  Q^H A
    void left(mat<S>& A, bool herm) const {
        const i64 k = i64(g.size());
        if (!herm)
            for (i64 j = k; j-- > 0;) hh_left(g[size_t(j)], g[size_t(j)].tau, A, 0);
        else
            for (i64 j = 0; j < k; ++j) hh_left(g[size_t(j)], cj(g[size_t(j)].tau), A, 0);
    }
    // A := A Q  or  A Q^H
    void right(mat<S>& A, bool herm) const {
        const i64 k = i64(g.size());
        if (!herm)
            for (i64 j = 0; j < k; ++j) hh_right(g[size_t(j)], g[size_t(j)].tau, A, A.r);
        else
            for (i64 j = k; j-- > 0;) hh_right(g[size_t(j)], cj(g[size_t(j)].tau), A, A.r);
    }
};

// xGEQR2: A = Q R, R overwrites A.
template <class S> ufac<S> geqr2(mat<S>& A) {
    const i64 m = A.r, n = A.c;
    if (m == 0 || n == 0) throw dim_err("qr: empty matrix");
    const i64 k = std::min(m, n);
    ufac<S> Q;
    Q.dim = m;
    Q.g.resize(size_t(k));
    vec<S> xb;
    for (i64 j = 0; j < k; ++j) {
        hh<S>& h = Q.g[size_t(j)];
        h.off = j;
        xb.assign(A.col(j) + j + 1, A.col(j) + m);
        const S beta = make_hh(A(j, j), xb.data(), m - j - 1, false, h);
        hh_left(h, cj(h.tau), A, j + 1);  // H^H applied
        A(j, j) = beta;
        for (i64 i = j + 1; i < m; ++i) A(i, j) = S(0);
    }
    return Q;
}

// xGERQ2 for any shape: rows bottom-up, reflectors from the right.  Returns
// Z with M_in = T Z (T overwrites M).
template <class S> ufac<S> gerq2(mat<S>& M) {
    const i64 r = M.r, c = M.c;
    if (r == 0 || c == 0) throw dim_err("rq: empty matrix");
    const i64 k = std::min(r, c);
    ufac<S> Z;
    Z.dim = c;
    Z.g.resize(size_t(k));
    vec<S> xb(static_cast<size_t>(c));
    for (i64 j = k; j-- > 0;) {
        const i64 row = r - k + j, pcol = c - k + j;
        hh<S>& h = Z.g[size_t(j)];
        h.off = 0;
        xb.resize(size_t(pcol));
        for (i64 t = 0; t < pcol; ++t) xb[size_t(t)] = cj(M(row, t));
        const S beta = make_hh(cj(M(row, pcol)), xb.data(), pcol, true, h);
        hh_right(h, h.tau, M, row);  // M := M H
        M(row, pcol) = beta;
        for (i64 t = 0; t < pcol; ++t) M(row, t) = S(0);
        h.tau = cj(h.tau);  // store G_j = H_j^H
    }
    return Z;
}

// ---- dense kernels ---------------------------------------------------------
template <class S> vec<S> mv(const mat<S>& A, const vec<S>& x, bool herm) {
    if (!herm) {
        if (i64(x.size()) != A.c) throw dim_err("gemv: x length != cols");
        vec<S> y(size_t(A.r), S(0));
        for (i64 j = 0; j < A.c; ++j) {
            const S xj = x[size_t(j)];
            const S* aj = A.col(j);
            for (i64 i = 0; i < A.r; ++i) y[size_t(i)] += xj * aj[i];
        }
        return y;
    }
    if (i64(x.size()) != A.r) throw dim_err("gemv: x length != rows");
    vec<S> y(size_t(A.c), S(0));
    for (i64 j = 0; j < A.c; ++j) {
        const S* aj = A.col(j);
        S s = S(0);
        for (i64 i = 0; i < A.r; ++i) s += cj(aj[i]) * x[size_t(i)];
        y[size_t(j)] = s;
    }
    return y;
}

template <class S>
vec<S> mv_blk(const mat<S>& M, i64 r0, i64 rows, i64 c0, i64 cols, const vec<S>& x, bool herm) {
    if (r0 + rows > M.r || c0 + cols > M.c) throw dim_err("gemv_sub: block out of range");
    if (!herm) {
        if (i64(x.size()) != cols) throw dim_err("gemv_sub: x length mismatch");
        vec<S> y(size_t(rows), S(0));
        for (i64 j = 0; j < cols; ++j) {
            const S xj = x[size_t(j)];
            const S* aj = M.col(c0 + j) + r0;
            for (i64 i = 0; i < rows; ++i) y[size_t(i)] += xj * aj[i];
        }
        return y;
    }
    if (i64(x.size()) != rows) throw dim_err("gemv_sub: x length mismatch");
    vec<S> y(size_t(cols), S(0));
    for (i64 j = 0; j < cols; ++j) {
        const S* aj = M.col(c0 + j) + r0;
        S s = S(0);
        for (i64 i = 0; i < rows; ++i) s += cj(aj[i]) * x[size_t(i)];
        y[size_t(j)] = s;
    }
    return y;
}

// upper-triangular block solve: N = column sweep, H = dot sweep
template <class S> vec<S> tri_blk(const mat<S>& M, i64 r0, i64 c0, i64 k, vec<S> x, bool herm) {
    if (r0 + k > M.r || c0 + k > M.c) throw dim_err("trsv_sub: block out of range");
    if (i64(x.size()) != k) throw dim_err("trsv_sub: rhs length mismatch");
    if (!herm) {
        for (i64 jj = k; jj-- > 0;) {
            const S piv = M(r0 + jj, c0 + jj);
            if (piv == S(0)) throw zero_pivot(jj);
            const S xj = x[size_t(jj)] / piv;
            x[size_t(jj)] = xj;
            const S* cjj = M.col(c0 + jj) + r0;
            for (i64 i = 0; i < jj; ++i) x[size_t(i)] -= xj * cjj[i];
        }
    } else {
        for (i64 j = 0; j < k; ++j) {
            const S piv = M(r0 + j, c0 + j);
            if (piv == S(0)) throw zero_pivot(j);
            const S* cjj = M.col(c0 + j) + r0;
            S s = x[size_t(j)];
            for (i64 i = 0; i < j; ++i) s -= cj(cjj[i]) * x[size_t(i)];
            x[size_t(j)] = s / cj(piv);
        }
    }
    return x;
}
template <class S> vec<S> tri(const mat<S>& R, const vec<S>& b, bool herm) {
    if (R.r != R.c) throw dim_err("trsv: matrix not square");
    return tri_blk(R, 0, 0, R.r, b, herm);
}

// double-double helpers (precision.hpp:131-142)
inline void two_sum(double a, double b, double& s, double& e) {
    s = a + b;
    const double z = s - a;
    e = (a - (s - z)) + (b - z);
}
inline void two_prod(double a, double b, double& p, double& e) {
    p = a * b;
    e = std::fma(a, b, -p);
}
inline double dd_dot(const double* x, i64 sx, const double* y, i64 n) {
    double s = 0.0, c = 0.0;
    for (i64 i = 0; i < n; ++i) {
        double p, pe, se;
        two_prod(x[i * sx], y[i], p, pe);
        two_sum(s, p, s, se);
        c += se + pe;
    }
    return s + c;
}

// ---- generalized factorizations -------------------------------------------
// GRQ: B = [0 R] Q,  A = Z T Q   (factor.hpp:34-52)
template <class S> struct grq_t {
    i64 m = 0, n = 0, p = 0;
    ufac<S> Q, Z;
    mat<S> R, T;
};
template <class S> grq_t<S> grq(const mat<S>& B, const mat<S>& A) {
    const i64 p = B.r, n = B.c, m = A.r;
    if (A.c != n) throw dim_err("grq: column counts differ");
    if (p > n || n > m + p) throw dim_err("grq: requires p <= n <= m + p");
    if (p == 0 || n == 0) throw dim_err("rq: empty matrix");
    grq_t<S> f;
    f.m = m;
    f.n = n;
    f.p = p;
    mat<S> Bw = B;
    f.Q = gerq2(Bw);
    f.R = mat<S>(p, p);
    for (i64 j = 0; j < p; ++j)
        for (i64 i = 0; i <= j; ++i) f.R(i, j) = Bw(i, n - p + j);
    mat<S> C = A;
    f.Q.right(C, true);
    f.Z = geqr2(C);
    f.T = std::move(C);
    return f;
}
// GQR: W = Q [R; 0],  V = Q T Z   (factor.hpp:55-75)
template <class S> struct gqr_t {
    i64 n = 0, m = 0, p = 0;
    ufac<S> Q, Z;
    mat<S> R, T;
};
template <class S> gqr_t<S> gqr(const mat<S>& W, const mat<S>& V) {
    const i64 n = W.r, m = W.c, p = V.c;
    if (V.r != n) throw dim_err("gqr: row counts differ");
    if (m > n || n > m + p) throw dim_err("gqr: requires m <= n <= m + p");
    gqr_t<S> f;
    f.n = n;
    f.m = m;
    f.p = p;
    mat<S> Ww = W;
    f.Q = geqr2(Ww);
    f.R = mat<S>(m, m);
    for (i64 j = 0; j < m; ++j)
        for (i64 i = 0; i <= j; ++i) f.R(i, j) = Ww(i, j);
    mat<S> C = V;
    f.Q.left(C, true);
    f.Z = gerq2(C);
    f.T = std::move(C);
    return f;
}

template <class To, class From> ufac<To> cast_f(const ufac<From>& Q) {
    ufac<To> o;
    o.dim = Q.dim;
    o.g.resize(Q.g.size());
    for (size_t j = 0; j < Q.g.size(); ++j) {
        o.g[j].off = Q.g[j].off;
        o.g[j].tau = cast<To>(Q.g[j].tau);
        o.g[j].v = cast_v<To>(Q.g[j].v);
    }
    return o;
}
template <class To, class From> grq_t<To> widen(const grq_t<From>& f) {
    grq_t<To> g;
    g.m = f.m;
    g.n = f.n;
    g.p = f.p;
    g.Q = cast_f<To>(f.Q);
    g.Z = cast_f<To>(f.Z);
    g.R = cast_m<To>(f.R);
    g.T = cast_m<To>(f.T);
    return g;
}
template <class To, class From> gqr_t<To> widen(const gqr_t<From>& f) {
    gqr_t<To> g;
    g.n = f.n;
    g.m = f.m;
    g.p = f.p;
    g.Q = cast_f<To>(f.Q);
    g.Z = cast_f<To>(f.Z);
    g.R = cast_m<To>(f.R);
    g.T = cast_m<To>(f.T);
    return g;
}

// ---- LSE -------------------------------------------------------------------
template <class S> struct lse_pb {
    mat<S> A, B;
    vec<S> b, d;
    void check() const {
        const i64 m = A.r, n = A.c, p = B.r;
        if (m == 0 || n == 0 || p == 0 || B.c == 0) throw dim_err("lse_problem: empty matrix");
        if (B.c != n) throw dim_err("lse_problem: column counts differ");
        if (p > n || n > m + p) throw dim_err("lse_problem: requires p <= n <= m + p");
        if (i64(b.size()) != m || i64(d.size()) != p) throw dim_err("lse_problem: rhs length");
    }
};

// null-space solve (lse.hpp:48-65)
template <class S> vec<S> lse_x(const grq_t<S>& f, const vec<S>& b, const vec<S>& d) {
    const i64 n = f.n, p = f.p;
    if (i64(b.size()) != f.m || i64(d.size()) != p) throw dim_err("lse_direct: rhs length");
    vec<S> y2 = tri(f.R, d, false);
    vec<S> c = f.Z.times(b, true);
    vec<S> rhs(c.begin(), c.begin() + (n - p));
    if (p > 0) {
        vec<S> t = mv_blk(f.T, 0, n - p, n - p, p, y2, false);
        for (i64 i = 0; i < n - p; ++i) rhs[size_t(i)] -= t[size_t(i)];
    }
    vec<S> y1 = tri_blk(f.T, 0, 0, n - p, rhs, false);
    vec<S> y(static_cast<size_t>(n));
    std::copy(y1.begin(), y1.end(), y.begin());
    std::copy(y2.begin(), y2.end(), y.begin() + (n - p));
    return f.Q.times(y, true);
}

// cascade of Algorithm 1 (lse.hpp:83-128)
template <class S>
void lse_corr(const grq_t<S>& f, const vec<S>& f1, const vec<S>& f2, const vec<S>& f3, vec<S>& dr,
              vec<S>& dv, vec<S>& dx) {
    const i64 m = f.m, n = f.n, p = f.p;
    if (i64(f1.size()) != m || i64(f2.size()) != p || i64(f3.size()) != n)
        throw dim_err("lse_correction_solve: rhs length");
    const i64 k = n - p;
    vec<S> u = f.Q.times(f3, false);
    vec<S> w = f.Z.times(f1, true);
    vec<S> y2 = tri(f.R, f2, false);
    vec<S> q1 = tri_blk(f.T, 0, 0, k, vec<S>(u.begin(), u.begin() + k), true);
    vec<S> rhs(static_cast<size_t>(k));
    {
        vec<S> t = mv_blk(f.T, 0, k, k, p, y2, false);
        for (i64 i = 0; i < k; ++i) rhs[size_t(i)] = w[size_t(i)] - q1[size_t(i)] - t[size_t(i)];
    }
    vec<S> y1 = tri_blk(f.T, 0, 0, k, rhs, false);
    vec<S> q(static_cast<size_t>(m));
    std::copy(q1.begin(), q1.end(), q.begin());
    {
        vec<S> t = mv_blk(f.T, k, m - k, k, p, y2, false);
        for (i64 i = k; i < m; ++i) q[size_t(i)] = w[size_t(i)] - t[size_t(i - k)];
    }
    dr = f.Z.times(q, false);
    vec<S> y(static_cast<size_t>(n));
    std::copy(y1.begin(), y1.end(), y.begin());
    std::copy(y2.begin(), y2.end(), y.begin() + k);
    dx = f.Q.times(y, true);
    vec<S> s = mv_blk(f.T, 0, k, k, p, q1, true);
    {
        vec<S> q2(q.begin() + k, q.end());
        vec<S> t = mv_blk(f.T, k, m - k, k, p, q2, true);
        for (i64 i = 0; i < p; ++i) s[size_t(i)] += t[size_t(i)] - u[size_t(k + i)];
    }
    dv = tri(f.R, s, true);
}

// v from R^H v = (Q A^H r)(n-p:n) (lse.hpp:156-173)
template <class W, class F>
vec<W> lse_v(const grq_t<F>& f, const mat<W>& A, const vec<W>& r, int ur) {
    vec<W> g;
    if (ur == 2) {
        if constexpr (traits<W>::cplx) throw bad_input("extended residual is real-only");
        else {
            g.resize(size_t(A.c));
            for (i64 j = 0; j < A.c; ++j) g[size_t(j)] = dd_dot(A.col(j), 1, r.data(), A.r);
        }
    } else {
        g = mv(A, r, true);
    }
    if constexpr (std::is_same_v<W, F>) {
        f.Q.apply(g, false);
        vec<W> tail(g.begin() + (f.n - f.p), g.end());
        return tri(f.R, tail, true);
    } else {
        const double s = one_if_zero(amax(g));
        vec<F> gf(g.size());
        for (size_t i = 0; i < g.size(); ++i) gf[i] = cast<F>(g[i] / s);
        f.Q.apply(gf, false);
        vec<F> tail(gf.begin() + (f.n - f.p), gf.end());
        vec<F> vf = tri(f.R, tail, true);
        vec<W> out(vf.size());
        for (size_t i = 0; i < vf.size(); ++i) out[i] = s * cast<W>(vf[i]);
        return out;
    }
}

// f1 = b - r - A x, f2 = d - B x, f3 = B^H v - A^H r (lse.hpp:181-258)
template <class W>
void lse_res(const lse_pb<W>& pb, const vec<W>& x, const vec<W>& r, const vec<W>& v, int ur,
             vec<W>& f1, vec<W>& f2, vec<W>& f3) {
    const i64 m = pb.A.r, n = pb.A.c, p = pb.B.r;
    if (i64(x.size()) != n || i64(r.size()) != m || i64(v.size()) != p)
        throw dim_err("lse_residuals: state length");
    if (ur != 2) {
        vec<W> ax = mv(pb.A, x, false);
        f1.resize(size_t(m));
        for (i64 i = 0; i < m; ++i) f1[size_t(i)] = pb.b[size_t(i)] - r[size_t(i)] - ax[size_t(i)];
        vec<W> bx = mv(pb.B, x, false);
        f2.resize(size_t(p));
        for (i64 i = 0; i < p; ++i) f2[size_t(i)] = pb.d[size_t(i)] - bx[size_t(i)];
        vec<W> atr = mv(pb.A, r, true);
        vec<W> btv = mv(pb.B, v, true);
        f3.resize(size_t(n));
        for (i64 j = 0; j < n; ++j) f3[size_t(j)] = btv[size_t(j)] - atr[size_t(j)];
        return;
    }
    if constexpr (traits<W>::cplx) {
        throw bad_input("extended residual is real-only");
    } else {
        {
            vec<double> s(static_cast<size_t>(m)), c(static_cast<size_t>(m), 0.0);
            for (i64 i = 0; i < m; ++i) {
                double e;
                two_sum(pb.b[size_t(i)], -r[size_t(i)], s[size_t(i)], e);
                c[size_t(i)] = e;
            }
            for (i64 j = 0; j < n; ++j) {
                const double xj = x[size_t(j)];
                const double* aj = pb.A.col(j);
                for (i64 i = 0; i < m; ++i) {
                    double pr, pe, se;
                    two_prod(-aj[i], xj, pr, pe);
                    two_sum(s[size_t(i)], pr, s[size_t(i)], se);
                    c[size_t(i)] += se + pe;
                }
            }
            f1.resize(size_t(m));
            for (i64 i = 0; i < m; ++i) f1[size_t(i)] = s[size_t(i)] + c[size_t(i)];
        }
        {
            vec<double> s(pb.d), c(size_t(p), 0.0);
            for (i64 j = 0; j < n; ++j) {
                const double xj = x[size_t(j)];
                const double* bj = pb.B.col(j);
                for (i64 i = 0; i < p; ++i) {
                    double pr, pe, se;
                    two_prod(-bj[i], xj, pr, pe);
                    two_sum(s[size_t(i)], pr, s[size_t(i)], se);
                    c[size_t(i)] += se + pe;
                }
            }
            f2.resize(size_t(p));
            for (i64 i = 0; i < p; ++i) f2[size_t(i)] = s[size_t(i)] + c[size_t(i)];
        }
        f3.resize(size_t(n));
        for (i64 j = 0; j < n; ++j) {
            double s = 0.0, c = 0.0;
            const double* aj = pb.A.col(j);
            for (i64 i = 0; i < m; ++i) {
                double pr, pe, se;
                two_prod(-aj[i], r[size_t(i)], pr, pe);
                two_sum(s, pr, s, se);
                c += se + pe;
            }
            const double* bj = pb.B.col(j);
            for (i64 i = 0; i < p; ++i) {
                double pr, pe, se;
                two_prod(bj[i], v[size_t(i)], pr, pe);
                two_sum(s, pr, s, se);
                c += se + pe;
            }
            f3[size_t(j)] = s + c;
        }
    }
}

inline double ratio(double num, double den) {
    if (den > 0.0) return num / den;
    return num == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
}

// divergence: 1e4 x growth over the running minimum, or non-finite (refine.hpp:79-91)
struct diverge_watch {
    double best = std::numeric_limits<double>::infinity();
    bool hit(double s) {
        if (!std::isfinite(s)) return true;
        if (s < best) best = s;
        return s >= 1e4 * best && best > 0.0;
    }
};

struct cfg_t {
    double tol;
    i64 maxit;
    int uf, us, ur;
    void check() const {
        if (!(tol > 0.0)) throw bad_input("tol must be positive");
        if (maxit < 1) throw bad_input("maxit must be >= 1");
        // u_f >= u_s >= u (= working) >= u_r, by unit roundoff
        auto u = [](int c) { return c == 0 ? 0x1p-24 : (c == 2 ? 0x1p-106 : 0x1p-53); };
        if (uf < 0 || uf > 2 || us < 0 || us > 2 || ur < 0 || ur > 2)
            throw bad_input("precision code out of range");
        if (u(uf) < u(us) || u(us) < 0x1p-53 || 0x1p-53 < u(ur))
            throw bad_input("requires u_f >= u_s >= u >= u_r");
    }
};

struct trace_t {
    int status = 1;  // max_iterations
    i64 iters = 0;
    vec<double> hist;
    double ph[6] = {0, 0, 0, 0, 0, 0};
};

struct lap_clock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double lap() {
        auto now = std::chrono::steady_clock::now();
        double s = std::chrono::duration<double>(now - t0).count();
        t0 = now;
        return s;
    }
};

template <class W> using low_t = typename traits<W>::low;

// four-precision classical IR, Algorithm 2 (lse.hpp:303-429)
template <class W>
void mplse(const lse_pb<W>& pb, const cfg_t& cfg, vec<W>& xo, vec<W>& ro, vec<W>& vo, trace_t& tr) {
    using L = low_t<W>;
    pb.check();
    cfg.check();
    const i64 m = pb.A.r, n = pb.A.c, p = pb.B.r;
    const bool lowf = cfg.uf == 0, lows = cfg.us == 0;
    lap_clock sw;
    const double sA = lowf ? one_if_zero(amax(pb.A.a)) : 1.0;
    const double sB = lowf ? one_if_zero(amax(pb.B.a)) : 1.0;
    const double cb = lowf ? one_if_zero(amax(pb.b)) : 1.0;
    const double cdd = lowf ? sB * cb / sA : 1.0;
    lse_pb<W> pr;
    pr.A = pb.A;
    pr.B = pb.B;
    if (lowf) {
        for (W& t : pr.A.a) t /= sA;
        for (W& t : pr.B.a) t /= sB;
    }
    pr.b.resize(pb.b.size());
    for (size_t i = 0; i < pb.b.size(); ++i) pr.b[i] = pb.b[i] / cb;
    pr.d.resize(pb.d.size());
    for (size_t i = 0; i < pb.d.size(); ++i) pr.d[i] = pb.d[i] / cdd;
    if (!all_fin(pr.d)) throw bad_input("mplse: rhs scaling overflowed");
    tr.ph[5] += sw.lap();

    grq_t<L> Fl;
    grq_t<W> Fw;
    mat<L> Al, Bl;
    if (lowf) {
        Al = cast_m<L>(pr.A);
        Bl = cast_m<L>(pr.B);
        Fl = grq(Bl, Al);
        if (!lows) Fw = widen<W>(Fl);
    } else {
        Fw = grq(pr.B, pr.A);
    }
    tr.ph[0] += sw.lap();

    vec<W> x, r, v;
    if (lowf) {
        vec<L> bl = cast_v<L>(pr.b), dl = cast_v<L>(pr.d);
        vec<L> xl = lse_x(Fl, bl, dl);
        vec<L> axl = mv(Al, xl, false);
        vec<L> rl(static_cast<size_t>(m));
        for (i64 i = 0; i < m; ++i) rl[size_t(i)] = bl[size_t(i)] - axl[size_t(i)];
        x = cast_v<W>(xl);
        r = cast_v<W>(rl);
        v = lse_v(Fl, pr.A, r, cfg.ur);
    } else {
        x = lse_x(Fw, pr.b, pr.d);
        vec<W> ax = mv(pr.A, x, false);
        r.resize(size_t(m));
        for (i64 i = 0; i < m; ++i) r[size_t(i)] = pr.b[size_t(i)] - ax[size_t(i)];
        v = lse_v(Fw, pr.A, r, cfg.ur);
    }
    tr.ph[1] += sw.lap();

    const double nb = nrm2(pr.b), nd = nrm2(pr.d), nA = nrmF(pr.A), nB = nrmF(pr.B);
    tr.ph[5] += sw.lap();

    diverge_watch watch;
    for (i64 pass = 1; pass <= cfg.maxit; ++pass) {
        vec<W> f1, f2, f3;
        lse_res(pr, x, r, v, cfg.ur, f1, f2, f3);
        const double g1 = nrm2(f1), g2 = nrm2(f2), g3 = nrm2(f3);
        const double sr = nrm2(r), sv = nrm2(v), sx = nrm2(x);
        tr.hist.push_back(g1 * cb);
        tr.hist.push_back(g2 * cdd);
        tr.hist.push_back(g3 * sA * cb);
        tr.iters = pass;
        tr.ph[2] += sw.lap();
        const double tol = cfg.tol;
        if (g1 <= tol * (nb + sr + nA * sx) && g2 <= tol * (nd + nB * sx) &&
            g3 <= tol * (nA * sr + nB * sv)) {
            tr.status = 0;
            break;
        }
        const double smax = std::max({ratio(g1, nb + sr + nA * sx), ratio(g2, nd + nB * sx),
                                      ratio(g3, nA * sr + nB * sv)});
        if (watch.hit(smax)) {
            tr.status = 2;
            break;
        }
        vec<W> dr, dv, dx;
        if (lows) {
            const double sig = one_if_zero(std::max({amax(f1), amax(f2), amax(f3)}));
            auto dem = [&](const vec<W>& f) {
                vec<L> o(f.size());
                for (size_t i = 0; i < f.size(); ++i) o[i] = cast<L>(f[i] / sig);
                return o;
            };
            auto pro = [&](const vec<L>& f) {
                vec<W> o(f.size());
                for (size_t i = 0; i < f.size(); ++i) o[i] = sig * cast<W>(f[i]);
                return o;
            };
            vec<L> a, b2, c;
            lse_corr(Fl, dem(f1), dem(f2), dem(f3), a, b2, c);
            dr = pro(a);
            dv = pro(b2);
            dx = pro(c);
        } else {
            lse_corr(Fw, f1, f2, f3, dr, dv, dx);
        }
        for (i64 i = 0; i < m; ++i) r[size_t(i)] += dr[size_t(i)];
        for (i64 i = 0; i < p; ++i) v[size_t(i)] += dv[size_t(i)];
        for (i64 i = 0; i < n; ++i) x[size_t(i)] += dx[size_t(i)];
        tr.ph[3] += sw.lap();
        if (!all_fin(r) || !all_fin(v) || !all_fin(x)) {
            tr.status = 2;
            break;
        }
    }
    xo.resize(x.size());
    for (size_t i = 0; i < x.size(); ++i) xo[i] = (cb / sA) * x[i];
    ro.resize(r.size());
    for (size_t i = 0; i < r.size(); ++i) ro[i] = cb * r[i];
    vo.resize(v.size());
    for (size_t i = 0; i < v.size(); ++i) vo[i] = (sA * cb / sB) * v[i];
    tr.ph[5] += sw.lap();
}

// ---- GLS -------------------------------------------------------------------
template <class S> struct gls_pb {
    mat<S> W, V;
    vec<S> d;
    void check() const {
        const i64 n = W.r, m = W.c, p = V.c;
        if (n == 0 || m == 0 || V.r == 0 || p == 0) throw dim_err("gls_problem: empty matrix");
        if (V.r != n) throw dim_err("gls_problem: row counts differ");
        if (m > n || n > m + p) throw dim_err("gls_problem: requires m <= n <= m + p");
        if (i64(d.size()) != n) throw dim_err("gls_problem: rhs length");
    }
};

// Paige's solve (gls.hpp:47-65)
template <class S> void gls_xy(const gqr_t<S>& f, const vec<S>& d, vec<S>& x, vec<S>& y) {
    const i64 n = f.n, m = f.m, p = f.p;
    if (i64(d.size()) != n) throw dim_err("gls_direct: rhs length");
    const i64 k = p - n + m;
    vec<S> c = f.Q.times(d, true);
    vec<S> s2 = tri_blk(f.T, m, k, n - m, vec<S>(c.begin() + m, c.end()), false);
    vec<S> rhs(c.begin(), c.begin() + m);
    if (n > m) {
        vec<S> t = mv_blk(f.T, 0, m, k, n - m, s2, false);
        for (i64 i = 0; i < m; ++i) rhs[size_t(i)] -= t[size_t(i)];
    }
    x = tri(f.R, rhs, false);
    vec<S> s(size_t(p), S(0));
    std::copy(s2.begin(), s2.end(), s.begin() + k);
    y = f.Z.times(s, true);
}

// z with W^H z = 0, V^H z = y (gls.hpp:71-82)
template <class S> vec<S> gls_z(const gqr_t<S>& f, const vec<S>& y) {
    const i64 n = f.n, m = f.m, p = f.p;
    if (i64(y.size()) != p) throw dim_err("init_z: y length");
    const i64 k = p - n + m;
    vec<S> g = f.Z.times(y, false);
    vec<S> vv = tri_blk(f.T, m, k, n - m, vec<S>(g.begin() + k, g.end()), true);
    vec<S> zq(size_t(n), S(0));
    std::copy(vv.begin(), vv.end(), zq.begin() + m);
    return f.Q.times(zq, false);
}

// cascade of Algorithm 3 (gls.hpp:106-154)
template <class S>
void gls_corr(const gqr_t<S>& f, const vec<S>& f1, const vec<S>& f2, const vec<S>& f3, vec<S>& dy,
              vec<S>& dz, vec<S>& dx) {
    const i64 n = f.n, m = f.m, p = f.p;
    if (i64(f1.size()) != p || i64(f2.size()) != n || i64(f3.size()) != m)
        throw dim_err("gls_correction_solve: rhs length");
    const i64 k = p - n + m;
    vec<S> u = f.Q.times(f2, true);
    vec<S> w = f.Z.times(f1, false);
    vec<S> h1 = tri(f.R, f3, true);
    vec<S> g2 = tri_blk(f.T, m, k, n - m, vec<S>(u.begin() + m, u.end()), false);
    vec<S> rhs2(static_cast<size_t>(n - m));
    {
        vec<S> t = mv_blk(f.T, 0, m, k, n - m, h1, true);
        for (i64 i = 0; i < n - m; ++i) rhs2[size_t(i)] = w[size_t(k + i)] - g2[size_t(i)] - t[size_t(i)];
    }
    vec<S> h2 = tri_blk(f.T, m, k, n - m, rhs2, true);
    vec<S> g(static_cast<size_t>(p));
    {
        vec<S> t = mv_blk(f.T, 0, m, 0, k, h1, true);
        for (i64 i = 0; i < k; ++i) g[size_t(i)] = w[size_t(i)] - t[size_t(i)];
        std::copy(g2.begin(), g2.end(), g.begin() + k);
    }
    dy = f.Z.times(g, true);
    vec<S> h(static_cast<size_t>(n));
    std::copy(h1.begin(), h1.end(), h.begin());
    std::copy(h2.begin(), h2.end(), h.begin() + m);
    dz = f.Q.times(h, false);
    for (S& t : dz) t = -t;
    vec<S> rhs1(u.begin(), u.begin() + m);
    {
        vec<S> g1(g.begin(), g.begin() + k);
        vec<S> a = mv_blk(f.T, 0, m, 0, k, g1, false);
        vec<S> b = mv_blk(f.T, 0, m, k, n - m, g2, false);
        for (i64 i = 0; i < m; ++i) rhs1[size_t(i)] -= a[size_t(i)] + b[size_t(i)];
    }
    dx = tri(f.R, rhs1, false);
}

// f1 = V^H z - y, f2 = d - W x - V y, f3 = W^H z (gls.hpp:161-232)
template <class W>
void gls_res(const gls_pb<W>& pb, const vec<W>& x, const vec<W>& y, const vec<W>& z, int ur,
             vec<W>& f1, vec<W>& f2, vec<W>& f3) {
    const i64 n = pb.W.r, m = pb.W.c, p = pb.V.c;
    if (i64(x.size()) != m || i64(y.size()) != p || i64(z.size()) != n)
        throw dim_err("gls_residuals: state length");
    if (ur != 2) {
        vec<W> vtz = mv(pb.V, z, true);
        f1.resize(size_t(p));
        for (i64 j = 0; j < p; ++j) f1[size_t(j)] = vtz[size_t(j)] - y[size_t(j)];
        vec<W> wx = mv(pb.W, x, false), vy = mv(pb.V, y, false);
        f2.resize(size_t(n));
        for (i64 i = 0; i < n; ++i) f2[size_t(i)] = pb.d[size_t(i)] - wx[size_t(i)] - vy[size_t(i)];
        f3 = mv(pb.W, z, true);
        return;
    }
    if constexpr (traits<W>::cplx) {
        throw bad_input("extended residual is real-only");
    } else {
        f1.resize(size_t(p));
        for (i64 j = 0; j < p; ++j) {
            double s = -y[size_t(j)], c = 0.0;
            const double* vj = pb.V.col(j);
            for (i64 i = 0; i < n; ++i) {
                double pr, pe, se;
                two_prod(vj[i], z[size_t(i)], pr, pe);
                two_sum(s, pr, s, se);
                c += se + pe;
            }
            f1[size_t(j)] = s + c;
        }
        {
            vec<double> s(pb.d), c(size_t(n), 0.0);
            for (i64 j = 0; j < m; ++j) {
                const double xj = x[size_t(j)];
                const double* wj = pb.W.col(j);
                for (i64 i = 0; i < n; ++i) {
                    double pr, pe, se;
                    two_prod(-wj[i], xj, pr, pe);
                    two_sum(s[size_t(i)], pr, s[size_t(i)], se);
                    c[size_t(i)] += se + pe;
                }
            }
            for (i64 j = 0; j < p; ++j) {
                const double yj = y[size_t(j)];
                const double* vj = pb.V.col(j);
                for (i64 i = 0; i < n; ++i) {
                    double pr, pe, se;
                    two_prod(-vj[i], yj, pr, pe);
                    two_sum(s[size_t(i)], pr, s[size_t(i)], se);
                    c[size_t(i)] += se + pe;
                }
            }
            f2.resize(size_t(n));
            for (i64 i = 0; i < n; ++i) f2[size_t(i)] = s[size_t(i)] + c[size_t(i)];
        }
        f3.resize(size_t(m));
        for (i64 j = 0; j < m; ++j) {
            double s = 0.0, c = 0.0;
            const double* wj = pb.W.col(j);
            for (i64 i = 0; i < n; ++i) {
                double pr, pe, se;
                two_prod(wj[i], z[size_t(i)], pr, pe);
                two_sum(s, pr, s, se);
                c += se + pe;
            }
            f3[size_t(j)] = s + c;
        }
    }
}

// Algorithm 4 (gls.hpp:276-387)
template <class W>
void mpgls(const gls_pb<W>& pb, const cfg_t& cfg, vec<W>& xo, vec<W>& yo, vec<W>& zo, trace_t& tr) {
    using L = low_t<W>;
    pb.check();
    cfg.check();
    const i64 n = pb.W.r, m = pb.W.c, p = pb.V.c;
    const bool lowf = cfg.uf == 0, lows = cfg.us == 0;
    lap_clock sw;
    const double sW = lowf ? one_if_zero(amax(pb.W.a)) : 1.0;
    const double sV = lowf ? one_if_zero(amax(pb.V.a)) : 1.0;
    const double cdd = lowf ? one_if_zero(amax(pb.d)) : 1.0;
    gls_pb<W> pr;
    pr.W = pb.W;
    pr.V = pb.V;
    if (lowf) {
        for (W& t : pr.W.a) t /= sW;
        for (W& t : pr.V.a) t /= sV;
    }
    pr.d.resize(pb.d.size());
    for (size_t i = 0; i < pb.d.size(); ++i) pr.d[i] = pb.d[i] / cdd;
    tr.ph[5] += sw.lap();

    gqr_t<L> Fl;
    gqr_t<W> Fw;
    if (lowf) {
        Fl = gqr(cast_m<L>(pr.W), cast_m<L>(pr.V));
        if (!lows) Fw = widen<W>(Fl);
    } else {
        Fw = gqr(pr.W, pr.V);
    }
    tr.ph[0] += sw.lap();

    vec<W> x, y, z;
    if (lowf) {
        vec<L> dl = cast_v<L>(pr.d), xl, yl;
        gls_xy(Fl, dl, xl, yl);
        vec<L> zl = gls_z(Fl, yl);
        x = cast_v<W>(xl);
        y = cast_v<W>(yl);
        z = cast_v<W>(zl);
    } else {
        gls_xy(Fw, pr.d, x, y);
        z = gls_z(Fw, y);
    }
    tr.ph[1] += sw.lap();

    const double nd = nrm2(pr.d), nW = nrmF(pr.W), nV = nrmF(pr.V);
    tr.ph[5] += sw.lap();

    diverge_watch watch;
    for (i64 pass = 1; pass <= cfg.maxit; ++pass) {
        vec<W> f1, f2, f3;
        gls_res(pr, x, y, z, cfg.ur, f1, f2, f3);
        const double g1 = nrm2(f1), g2 = nrm2(f2), g3 = nrm2(f3);
        const double sx = nrm2(x), sy = nrm2(y), sz = nrm2(z);
        tr.hist.push_back(g1 * cdd / sV);
        tr.hist.push_back(g2 * cdd);
        tr.hist.push_back(g3 * sW * cdd / (sV * sV));
        tr.iters = pass;
        tr.ph[2] += sw.lap();
        const double tol = cfg.tol;
        if (g1 <= tol * (sy + nV * sz) && g2 <= tol * (nd + nW * sx + nV * sy) &&
            g3 <= tol * nW * sz) {
            tr.status = 0;
            break;
        }
        const double smax = std::max({ratio(g1, sy + nV * sz), ratio(g2, nd + nW * sx + nV * sy),
                                      ratio(g3, nW * sz)});
        if (watch.hit(smax)) {
            tr.status = 2;
            break;
        }
        vec<W> dy, dz, dx;
        if (lows) {
            const double sig = one_if_zero(std::max({amax(f1), amax(f2), amax(f3)}));
            auto dem = [&](const vec<W>& f) {
                vec<L> o(f.size());
                for (size_t i = 0; i < f.size(); ++i) o[i] = cast<L>(f[i] / sig);
                return o;
            };
            auto pro = [&](const vec<L>& f) {
                vec<W> o(f.size());
                for (size_t i = 0; i < f.size(); ++i) o[i] = sig * cast<W>(f[i]);
                return o;
            };
            vec<L> a, b2, c;
            gls_corr(Fl, dem(f1), dem(f2), dem(f3), a, b2, c);
            dy = pro(a);
            dz = pro(b2);
            dx = pro(c);
        } else {
            gls_corr(Fw, f1, f2, f3, dy, dz, dx);
        }
        for (i64 i = 0; i < m; ++i) x[size_t(i)] += dx[size_t(i)];
        for (i64 i = 0; i < p; ++i) y[size_t(i)] += dy[size_t(i)];
        for (i64 i = 0; i < n; ++i) z[size_t(i)] += dz[size_t(i)];
        tr.ph[3] += sw.lap();
        if (!all_fin(x) || !all_fin(y) || !all_fin(z)) {
            tr.status = 2;
            break;
        }
    }
    xo.resize(x.size());
    for (size_t i = 0; i < x.size(); ++i) xo[i] = (cdd / sW) * x[i];
    yo.resize(y.size());
    for (size_t i = 0; i < y.size(); ++i) yo[i] = (cdd / sV) * y[i];
    zo.resize(z.size());
    for (size_t i = 0; i < z.size(); ++i) zo[i] = (cdd / (sV * sV)) * z[i];
    tr.ph[5] += sw.lap();
}

// ---- seeded generator (generate.hpp:46-106 with random.hpp:16-30) ----------
inline mat<double> gauss_m(i64 r, i64 c, std::mt19937_64& g) {
    std::normal_distribution<double> nd(0.0, 1.0);
    mat<double> M(r, c);
    for (double& x : M.a) x = nd(g);
    return M;
}
inline vec<double> gauss_v(i64 n, std::mt19937_64& g) {
    std::normal_distribution<double> nd(0.0, 1.0);
    vec<double> v(static_cast<size_t>(n));
    for (double& x : v) x = nd(g);
    return v;
}
inline vec<double> sv_profile(i64 k, double cond, int dist) {
    vec<double> s(size_t(k), 1.0);
    if (k == 1) return s;
    for (i64 i = 0; i < k; ++i) {
        const double t = double(i) / double(k - 1);
        s[size_t(i)] = dist == 0 ? std::pow(cond, -t) : 1.0 - (1.0 - 1.0 / cond) * t;
    }
    return s;
}

// ---- C marshalling ---------------------------------------------------------
template <class S> mat<S> as_mat(const S* p, i64 r, i64 c) {
    mat<S> M(r, c);
    if (r * c) std::memcpy(M.a.data(), p, sizeof(S) * size_t(r * c));
    return M;
}
template <class S> vec<S> as_vec(const S* p, i64 n) { return vec<S>(p, p + n); }
template <class S> void out(const vec<S>& v, S* o) {
    if (o) std::copy(v.begin(), v.end(), o);
}

template <class Fn> int guard(Fn&& fn, int64_t* sing) {
    try {
        fn();
        return 0;
    } catch (const zero_pivot& e) {
        if (sing) *sing = e.idx;
        return 3;
    } catch (const dim_err&) {
        return 1;
    } catch (const bad_input&) {
        return 2;
    } catch (...) {
        return 9;
    }
}

inline void put_tr(const trace_t& t, int32_t* st, int64_t* it, double* hist, double* ph) {
    if (st) *st = t.status;
    if (it) *it = t.iters;
    if (hist) std::copy(t.hist.begin(), t.hist.end(), hist);
    if (ph)
        for (int i = 0; i < 6; ++i) ph[i] = t.ph[i];
}

}  // namespace port

using namespace port;

extern "C" {

int orc_mplse(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
              const double* b, const double* d, double tol, int64_t maxit, int uf, int us,
              int ur, double* x, double* r, double* v, int32_t* status, int64_t* iters,
              double* hist, double* phases, int64_t* sing) {
    return guard(
        [&] {
            lse_pb<double> pb{as_mat(A, m, n), as_mat(B, p, n), as_vec(b, m), as_vec(d, p)};
            vec<double> xo, ro, vo;
            trace_t tr;
            mplse(pb, cfg_t{tol, maxit, uf, us, ur}, xo, ro, vo, tr);
            out(xo, x);
            out(ro, r);
            out(vo, v);
            put_tr(tr, status, iters, hist, phases);
        },
        sing);
}

int orc_mpgls(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
              const double* d, double tol, int64_t maxit, int uf, int us, int ur, double* x,
              double* y, double* z, int32_t* status, int64_t* iters, double* hist,
              double* phases, int64_t* sing) {
    return guard(
        [&] {
            gls_pb<double> pb{as_mat(W, n, m), as_mat(V, n, p), as_vec(d, n)};
            vec<double> xo, yo, zo;
            trace_t tr;
            mpgls(pb, cfg_t{tol, maxit, uf, us, ur}, xo, yo, zo, tr);
            out(xo, x);
            out(yo, y);
            out(zo, z);
            put_tr(tr, status, iters, hist, phases);
        },
        sing);
}

// complex128 problems with complex64 factors (C5); arrays are interleaved (re, im)
int orc_mpgls_z(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                const double* d, double tol, int64_t maxit, int uf, int us, int ur, double* x,
                double* y, double* z, int32_t* status, int64_t* iters, double* hist,
                double* phases, int64_t* sing) {
    return guard(
        [&] {
            gls_pb<cd> pb{as_mat(reinterpret_cast<const cd*>(W), n, m),
                          as_mat(reinterpret_cast<const cd*>(V), n, p),
                          as_vec(reinterpret_cast<const cd*>(d), n)};
            vec<cd> xo, yo, zo;
            trace_t tr;
            mpgls(pb, cfg_t{tol, maxit, uf, us, ur}, xo, yo, zo, tr);
            out(xo, reinterpret_cast<cd*>(x));
            out(yo, reinterpret_cast<cd*>(y));
            out(zo, reinterpret_cast<cd*>(z));
            put_tr(tr, status, iters, hist, phases);
        },
        sing);
}

int orc_mplse_z(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                const double* b, const double* d, double tol, int64_t maxit, int uf, int us,
                int ur, double* x, double* r, double* v, int32_t* status, int64_t* iters,
                double* hist, double* phases, int64_t* sing) {
    return guard(
        [&] {
            lse_pb<cd> pb{as_mat(reinterpret_cast<const cd*>(A), m, n),
                          as_mat(reinterpret_cast<const cd*>(B), p, n),
                          as_vec(reinterpret_cast<const cd*>(b), m),
                          as_vec(reinterpret_cast<const cd*>(d), p)};
            vec<cd> xo, ro, vo;
            trace_t tr;
            mplse(pb, cfg_t{tol, maxit, uf, us, ur}, xo, ro, vo, tr);
            out(xo, reinterpret_cast<cd*>(x));
            out(ro, reinterpret_cast<cd*>(r));
            out(vo, reinterpret_cast<cd*>(v));
            put_tr(tr, status, iters, hist, phases);
        },
        sing);
}

int orc_mplse_batch(int64_t batch, int64_t m, int64_t n, int64_t p, const double* A,
                    const double* B, const double* b, const double* d, double tol,
                    int64_t maxit, int uf, int us, int ur, double* x, double* r, double* v,
                    int32_t* status, int64_t* iters, int32_t* err, int nthreads) {
    (void)nthreads;  // the port is the scalar (1-core) checker
    for (int64_t i = 0; i < batch; ++i) {
        int64_t sing = -1;
        const int rc = orc_mplse(m, n, p, A + i * m * n, B + i * p * n, b + i * m, d + i * p, tol,
                                 maxit, uf, us, ur, x ? x + i * n : nullptr, r ? r + i * m : nullptr,
                                 v ? v + i * p : nullptr, status ? status + i : nullptr,
                                 iters ? iters + i : nullptr, nullptr, nullptr, &sing);
        if (err) err[i] = rc;
    }
    return 0;
}

int orc_gen_lse(int64_t m, int64_t n, int64_t p, double cond, uint64_t seed, int dist,
                double* A, double* B, double* b, double* d) {
    return guard(
        [&] {
            if (!(cond >= 1.0)) throw bad_input("cond must be >= 1");
            if (m == 0 || n == 0 || p == 0) throw dim_err("zero dimension");
            if (p > n || n > m + p) throw dim_err("LSE requires p <= n <= m + p");
            std::mt19937_64 g(seed);
            mat<double> G1 = gauss_m(m + p, n, g);
            ufac<double> q1 = geqr2(G1);
            mat<double> G2 = gauss_m(n, n, g);
            ufac<double> q2 = geqr2(G2);
            vec<double> sv = sv_profile(n, cond, dist);
            mat<double> S(m + p, n);
            for (i64 i = 0; i < n; ++i) S(i, i) = sv[size_t(i)];
            q2.right(S, false);
            q1.left(S, false);
            for (i64 j = 0; j < n; ++j) {
                for (i64 i = 0; i < m; ++i) A[j * m + i] = S(i, j);
                for (i64 i = 0; i < p; ++i) B[j * p + i] = S(m + i, j);
            }
            out(gauss_v(m, g), b);
            out(gauss_v(p, g), d);
        },
        nullptr);
}

int orc_gen_gls(int64_t n, int64_t m, int64_t p, double cond, uint64_t seed, int dist,
                double* W, double* V, double* d) {
    return guard(
        [&] {
            if (!(cond >= 1.0)) throw bad_input("cond must be >= 1");
            if (m == 0 || n == 0 || p == 0) throw dim_err("zero dimension");
            if (m > n || n > m + p) throw dim_err("GLS requires m <= n <= m + p");
            std::mt19937_64 g(seed);
            mat<double> G1 = gauss_m(n, n, g);
            ufac<double> q1 = geqr2(G1);
            mat<double> G2 = gauss_m(m + p, n, g);
            ufac<double> q2 = geqr2(G2);
            vec<double> sv = sv_profile(n, cond, dist);
            mat<double> S(n, m + p);
            for (i64 i = 0; i < n; ++i) S(i, i) = sv[size_t(i)];
            q2.right(S, true);
            q1.left(S, false);
            for (i64 i = 0; i < n; ++i) {
                for (i64 j = 0; j < m; ++j) W[j * n + i] = S(i, j);
                for (i64 j = 0; j < p; ++j) V[j * n + i] = S(i, m + j);
            }
            out(gauss_v(n, g), d);
        },
        nullptr);
}

int orc_lse_residuals(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                      const double* b, const double* d, const double* x, const double* r,
                      const double* v, int ur, double* f1, double* f2, double* f3) {
    return guard(
        [&] {
            lse_pb<double> pb{as_mat(A, m, n), as_mat(B, p, n), as_vec(b, m), as_vec(d, p)};
            vec<double> a, b2, c;
            lse_res(pb, as_vec(x, n), as_vec(r, m), as_vec(v, p), ur, a, b2, c);
            out(a, f1);
            out(b2, f2);
            out(c, f3);
        },
        nullptr);
}

int orc_gls_residuals(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                      const double* d, const double* x, const double* y, const double* z,
                      int ur, double* f1, double* f2, double* f3) {
    return guard(
        [&] {
            gls_pb<double> pb{as_mat(W, n, m), as_mat(V, n, p), as_vec(d, n)};
            vec<double> a, b2, c;
            gls_res(pb, as_vec(x, m), as_vec(y, p), as_vec(z, n), ur, a, b2, c);
            out(a, f1);
            out(b2, f2);
            out(c, f3);
        },
        nullptr);
}

int orc_lse_correction(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                       const double* f1, const double* f2, const double* f3, int uf,
                       double* dr, double* dv, double* dx, int64_t* sing) {
    return guard(
        [&] {
            mat<double> Am = as_mat(A, m, n), Bm = as_mat(B, p, n);
            vec<double> g1 = as_vec(f1, m), g2 = as_vec(f2, p), g3 = as_vec(f3, n);
            if (uf == 0) {
                auto F = grq(cast_m<float>(Bm), cast_m<float>(Am));
                vec<float> a, b2, c;
                lse_corr(F, cast_v<float>(g1), cast_v<float>(g2), cast_v<float>(g3), a, b2, c);
                out(cast_v<double>(a), dr);
                out(cast_v<double>(b2), dv);
                out(cast_v<double>(c), dx);
            } else {
                auto F = grq(Bm, Am);
                vec<double> a, b2, c;
                lse_corr(F, g1, g2, g3, a, b2, c);
                out(a, dr);
                out(b2, dv);
                out(c, dx);
            }
        },
        sing);
}

int orc_gls_correction(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                       const double* f1, const double* f2, const double* f3, int uf,
                       double* dy, double* dz, double* dx, int64_t* sing) {
    return guard(
        [&] {
            mat<double> Wm = as_mat(W, n, m), Vm = as_mat(V, n, p);
            vec<double> g1 = as_vec(f1, p), g2 = as_vec(f2, n), g3 = as_vec(f3, m);
            if (uf == 0) {
                auto F = gqr(cast_m<float>(Wm), cast_m<float>(Vm));
                vec<float> a, b2, c;
                gls_corr(F, cast_v<float>(g1), cast_v<float>(g2), cast_v<float>(g3), a, b2, c);
                out(cast_v<double>(a), dy);
                out(cast_v<double>(b2), dz);
                out(cast_v<double>(c), dx);
            } else {
                auto F = gqr(Wm, Vm);
                vec<double> a, b2, c;
                gls_corr(F, g1, g2, g3, a, b2, c);
                out(a, dy);
                out(b2, dz);
                out(c, dx);
            }
        },
        sing);
}

int orc_lse_direct(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                   const double* b, const double* d, double* x, double* r, double* v,
                   int64_t* sing) {
    // lse.hpp:132-152: x by the null-space method, r = b - Z T Q x, R^T v = (T^T Z^T r)(n-p:n)
    return guard(
        [&] {
            mat<double> Am = as_mat(A, m, n), Bm = as_mat(B, p, n);
            vec<double> bv = as_vec(b, m), dv = as_vec(d, p);
            auto F = grq(Bm, Am);
            vec<double> xs = lse_x(F, bv, dv);
            vec<double> qx = F.Q.times(xs, false);
            vec<double> tqx = mv(F.T, qx, false);
            F.Z.apply(tqx, false);
            vec<double> rs(static_cast<size_t>(m));
            for (i64 i = 0; i < m; ++i) rs[size_t(i)] = bv[size_t(i)] - tqx[size_t(i)];
            vec<double> ztr = F.Z.times(rs, true);
            vec<double> ttz = mv(F.T, ztr, true);
            vec<double> tail(ttz.begin() + (n - p), ttz.end());
            out(xs, x);
            out(rs, r);
            out(tri(F.R, tail, true), v);
        },
        sing);
}

int orc_gls_direct(int64_t n, int64_t m, int64_t p, const double* W, const double* V,
                   const double* d, double* x, double* y, double* z, int64_t* sing) {
    return guard(
        [&] {
            auto F = gqr(as_mat(W, n, m), as_mat(V, n, p));
            vec<double> xs, ys;
            gls_xy(F, as_vec(d, n), xs, ys);
            out(xs, x);
            out(ys, y);
            out(gls_z(F, ys), z);
        },
        sing);
}

double orc_extended_dot(int64_t n, const double* x, const double* y) { return dd_dot(x, 1, y, n); }

int orc_trsv(int64_t n, const double* T, const double* rhs, int transpose, double* x,
             int64_t* sing) {
    return guard([&] { out(tri(as_mat(T, n, n), as_vec(rhs, n), transpose != 0), x); }, sing);
}

}  // extern "C"
