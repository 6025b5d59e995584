// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Stand-ins for the Eigen arithmetic the reference calls on the compress path
// (sthosvd.cpp:78-99,160-162): triangular Gram, SelfAdjointEigenSolver
// (Householder tridiagonalisation + implicit symmetric QR with Wilkinson
// shift, ascending sort), thin SVD for rows > cols (one-sided Jacobi in place
// of BDCSVD), the row-major transpose (tensor.cpp:105-144) and the reductions
// of kernels*.cpp.  Parity for these is by tolerance (Eigen is absent here).
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

#include "orc.hpp"

namespace orc {

std::size_t numel(const Shape& s) {
    std::size_t n = 1;
    for (auto v : s) n *= v;
    return n;
}

std::vector<std::size_t> strides_of(const Shape& s) {
    std::vector<std::size_t> st(s.size());
    std::size_t acc = 1;
    for (std::size_t i = s.size(); i-- > 0;) {
        st[i] = acc;
        acc *= s[i];
    }
    return st;
}

bool valid_perm(const Perm& p) {
    std::vector<bool> seen(p.size(), false);
    for (auto v : p) {
        if (v >= p.size() || seen[v]) return false;
        seen[v] = true;
    }
    return true;
}

Perm inverse_perm(const Perm& p) {
    Perm q(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) q[p[i]] = i;
    return q;
}

Perm stable_ascending(const Shape& s) {
    Perm p(s.size());
    std::iota(p.begin(), p.end(), std::size_t{0});
    std::stable_sort(p.begin(), p.end(), [&](std::size_t a, std::size_t b) { return s[a] < s[b]; });
    return p;
}

template <class T>
std::vector<T> permute_axes(const std::vector<T>& src, const Shape& shape, const Perm& p) {
    const std::size_t d = shape.size();
    if (p.size() != d || !valid_perm(p)) throw Error("transpose: invalid permutation");
    Shape out(d);
    for (std::size_t i = 0; i < d; ++i) out[i] = shape[p[i]];
    const auto in_st = strides_of(shape);
    std::vector<std::size_t> g(d);
    for (std::size_t i = 0; i < d; ++i) g[i] = in_st[p[i]];
    std::vector<T> dst(src.size());
    std::vector<std::size_t> idx(d, 0);
    std::size_t off = 0;
    for (std::size_t o = 0; o < dst.size(); ++o) {
        dst[o] = src[off];
        for (std::size_t m = d; m-- > 0;) {  // odometer, last output axis fastest
            off += g[m];
            if (++idx[m] < out[m]) break;
            off -= out[m] * g[m];
            idx[m] = 0;
        }
    }
    return dst;
}
template std::vector<float> permute_axes(const std::vector<float>&, const Shape&, const Perm&);
template std::vector<double> permute_axes(const std::vector<double>&, const Shape&, const Perm&);

// ---- reductions: lane-for-lane restatement of the AVX2 backend's summation
// order (kernels_avx2.cpp:128-160): 8 (fp64) / 4 (fp32) fused accumulators,
// pairwise horizontal add, fused scalar tail.
double sum_sq(const double* x, std::size_t n) {
    double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::size_t i = 0;
    for (; i + 8 <= n; i += 8)
        for (int l = 0; l < 8; ++l) a[l] = std::fma(x[i + l], x[i + l], a[l]);
    double v[4];
    for (int l = 0; l < 4; ++l) v[l] = a[l] + a[l + 4];
    double s = (v[0] + v[2]) + (v[1] + v[3]);
    for (; i < n; ++i) s = std::fma(x[i], x[i], s);
    return s;
}

double sum_sq(const float* x, std::size_t n) {
    double a[4] = {0, 0, 0, 0};
    std::size_t i = 0;
    for (; i + 4 <= n; i += 4)
        for (int l = 0; l < 4; ++l) {
            const double v = x[i + l];
            a[l] = std::fma(v, v, a[l]);
        }
    double s = (a[0] + a[2]) + (a[1] + a[3]);
    for (; i < n; ++i) {
        const double v = x[i];
        s = std::fma(v, v, s);
    }
    return s;
}

double max_abs_d(const double* x, std::size_t n) {
    double m = 0;
    for (std::size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(x[i]));
    return m;
}
float max_abs_f(const float* x, std::size_t n) {
    float m = 0;
    for (std::size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(x[i]));
    return m;
}
template <class T>
bool finite_all(const T* x, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i)
        if (!std::isfinite(x[i])) return false;
    return true;
}
template bool finite_all(const float*, std::size_t);
template bool finite_all(const double*, std::size_t);

// ---- symmetric eigensolver -------------------------------------------------
namespace {

template <class T>
void givens(T p, T q, T& c, T& s) {  // G^T [p; q] = [r; 0], G = [c s; -s c]
    if (q == T(0)) {
        c = p < T(0) ? T(-1) : T(1);
        s = T(0);
    } else if (p == T(0)) {
        c = T(0);
        s = q < T(0) ? T(1) : T(-1);
    } else if (std::fabs(p) > std::fabs(q)) {
        const T t = q / p;
        T u = std::sqrt(T(1) + t * t);
        if (p < T(0)) u = -u;
        c = T(1) / u;
        s = -t * c;
    } else {
        const T t = p / q;
        T u = std::sqrt(T(1) + t * t);
        if (q < T(0)) u = -u;
        s = -T(1) / u;
        c = -t * s;
    }
}

}  // namespace

// a: column-major n x n, lower triangle significant. On return a holds the
// eigenvectors (columns) and evals the ascending eigenvalues.
template <class T>
void sym_eig(std::vector<T>& a, std::size_t n, std::vector<T>& evals) {
    auto A = [&](std::size_t i, std::size_t j) -> T& { return a[i + j * n]; };
    for (std::size_t j = 0; j < n; ++j)
        for (std::size_t i = 0; i < j; ++i) A(i, j) = A(j, i);
    T scale = 0;
    for (auto v : a) scale = std::max(scale, std::fabs(v));
    if (scale == T(0)) scale = T(1);
    for (auto& v : a) v /= scale;

    // Householder tridiagonalisation, Q accumulated explicitly.
    std::vector<T> q(n * n, T(0));
    for (std::size_t i = 0; i < n; ++i) q[i + i * n] = T(1);
    std::vector<T> d(n), e(n > 0 ? n - 1 : 0), v(n), w(n);
    for (std::size_t k = 0; k + 2 < n; ++k) {
        const std::size_t m = n - k - 1;  // length of the vector below the diagonal
        T alpha = 0;
        for (std::size_t i = k + 1; i < n; ++i) alpha += A(i, k) * A(i, k);
        alpha = std::sqrt(alpha);
        if (alpha == T(0)) continue;
        const T x0 = A(k + 1, k);
        const T beta = x0 >= T(0) ? -alpha : alpha;  // new subdiagonal entry
        for (std::size_t i = 0; i < m; ++i) v[i] = A(k + 1 + i, k);
        v[0] -= beta;
        T vn = 0;
        for (std::size_t i = 0; i < m; ++i) vn += v[i] * v[i];
        if (vn == T(0)) continue;
        const T tau = T(2) / vn;  // H = I - tau v v^T
        // w = tau * A22 v ; A22 <- A22 - v w^T - w v^T + (tau/... ) symmetric update
        for (std::size_t i = 0; i < m; ++i) {
            T s = 0;
            for (std::size_t j = 0; j < m; ++j) s += A(k + 1 + i, k + 1 + j) * v[j];
            w[i] = tau * s;
        }
        T vw = 0;
        for (std::size_t i = 0; i < m; ++i) vw += v[i] * w[i];
        const T half = T(0.5) * tau * vw;
        for (std::size_t i = 0; i < m; ++i) w[i] -= half * v[i];
        for (std::size_t j = 0; j < m; ++j)
            for (std::size_t i = 0; i < m; ++i)
                A(k + 1 + i, k + 1 + j) -= v[i] * w[j] + w[i] * v[j];
        A(k + 1, k) = beta;
        A(k, k + 1) = beta;
        for (std::size_t i = k + 2; i < n; ++i) A(i, k) = A(k, i) = T(0);
        // Q <- Q H  (columns k+1..n-1)
        for (std::size_t r = 0; r < n; ++r) {
            T s = 0;
            for (std::size_t i = 0; i < m; ++i) s += q[r + (k + 1 + i) * n] * v[i];
            s *= tau;
            for (std::size_t i = 0; i < m; ++i) q[r + (k + 1 + i) * n] -= s * v[i];
        }
    }
    for (std::size_t i = 0; i < n; ++i) d[i] = A(i, i);
    for (std::size_t i = 0; i + 1 < n; ++i) e[i] = A(i + 1, i);

    // implicit symmetric QR with Wilkinson shift
    const T eps = std::numeric_limits<T>::epsilon();
    const T tiny = std::numeric_limits<T>::min();
    std::ptrdiff_t end = static_cast<std::ptrdiff_t>(n) - 1;
    std::size_t iter = 0;
    while (end > 0) {
        for (std::ptrdiff_t i = 0; i < end; ++i) {
            if (std::fabs(e[i]) < tiny || std::fabs(e[i]) <= eps * (std::fabs(d[i]) + std::fabs(d[i + 1])))
                e[i] = T(0);
        }
        while (end > 0 && e[end - 1] == T(0)) --end;
        if (end <= 0) break;
        if (++iter > 30 * n) throw Error("sthosvd: eigendecomposition failed");
        std::ptrdiff_t start = end - 1;
        while (start > 0 && e[start - 1] != T(0)) --start;
        const T td = (d[end - 1] - d[end]) * T(0.5);
        const T ee = e[end - 1];
        T mu = d[end];
        if (td == T(0)) {
            mu -= std::fabs(ee);
        } else {
            const T h = std::hypot(td, ee);
            mu -= (ee * ee) / (td + (td > T(0) ? h : -h));
        }
        T x = d[start] - mu, z = e[start];
        for (std::ptrdiff_t k = start; k < end && z != T(0); ++k) {
            T c, s;
            givens(x, z, c, s);
            const T sdk = s * d[k] + c * e[k];
            const T dkp1 = s * e[k] + c * d[k + 1];
            d[k] = c * (c * d[k] - s * e[k]) - s * (c * e[k] - s * d[k + 1]);
            d[k + 1] = s * sdk + c * dkp1;
            e[k] = c * sdk - s * dkp1;
            if (k > start) e[k - 1] = c * e[k - 1] - s * z;
            x = e[k];
            if (k < end - 1) {
                z = -s * e[k + 1];
                e[k + 1] = c * e[k + 1];
            }
            for (std::size_t r = 0; r < n; ++r) {
                const T a0 = q[r + k * n], a1 = q[r + (k + 1) * n];
                q[r + k * n] = c * a0 - s * a1;
                q[r + (k + 1) * n] = s * a0 + c * a1;
            }
        }
    }
    // ascending selection sort, columns follow
    for (std::size_t i = 0; i + 1 < n; ++i) {
        std::size_t km = i;
        for (std::size_t j = i + 1; j < n; ++j)
            if (d[j] < d[km]) km = j;
        if (km != i) {
            std::swap(d[i], d[km]);
            for (std::size_t r = 0; r < n; ++r) std::swap(q[r + i * n], q[r + km * n]);
        }
    }
    evals.resize(n);
    for (std::size_t i = 0; i < n; ++i) evals[i] = d[i] * scale;
    a = std::move(q);
}
template void sym_eig(std::vector<float>&, std::size_t, std::vector<float>&);
template void sym_eig(std::vector<double>&, std::size_t, std::vector<double>&);

// ---- thin SVD (rows > cols) by one-sided Jacobi on the columns --------------
template <class T>
void thin_svd(const T* b, std::size_t rows, std::size_t cols, std::vector<T>& u, std::vector<T>& sv) {
    std::vector<double> w(rows * cols);  // column-major working copy, in double
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) w[i + j * rows] = static_cast<double>(b[i * cols + j]);
    auto col = [&](std::size_t j) { return w.data() + j * rows; };
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0;
        for (std::size_t p = 0; p + 1 < cols; ++p)
            for (std::size_t q = p + 1; q < cols; ++q) {
                double al = 0, be = 0, ga = 0;
                const double* x = col(p);
                const double* y = col(q);
                for (std::size_t i = 0; i < rows; ++i) {
                    al += x[i] * x[i];
                    be += y[i] * y[i];
                    ga += x[i] * y[i];
                }
                if (ga == 0.0 || std::fabs(ga) <= 1e-17 * std::sqrt(al * be)) continue;
                off = std::max(off, std::fabs(ga) / std::sqrt(al * be));
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                double* xm = col(p);
                double* ym = col(q);
                for (std::size_t i = 0; i < rows; ++i) {
                    const double xi = xm[i], yi = ym[i];
                    xm[i] = c * xi - s * yi;
                    ym[i] = s * xi + c * yi;
                }
            }
        if (off < 1e-15) break;
    }
    std::vector<double> nrm(cols);
    for (std::size_t j = 0; j < cols; ++j) {
        double s = 0;
        for (std::size_t i = 0; i < rows; ++i) s += col(j)[i] * col(j)[i];
        nrm[j] = std::sqrt(s);
    }
    std::vector<std::size_t> ord(cols);
    std::iota(ord.begin(), ord.end(), std::size_t{0});
    std::stable_sort(ord.begin(), ord.end(), [&](auto a2, auto b2) { return nrm[a2] > nrm[b2]; });
    std::vector<double> ud(rows * cols, 0.0);
    sv.resize(cols);
    for (std::size_t jj = 0; jj < cols; ++jj) {
        const std::size_t j = ord[jj];
        sv[jj] = static_cast<T>(nrm[j]);
        double* dst = ud.data() + jj * rows;
        if (nrm[j] > 0)
            for (std::size_t i = 0; i < rows; ++i) dst[i] = col(j)[i] / nrm[j];
    }
    // complete null columns to an orthonormal set (Gram-Schmidt against e_i)
    for (std::size_t jj = 0; jj < cols; ++jj) {
        double* dst = ud.data() + jj * rows;
        double nn = 0;
        for (std::size_t i = 0; i < rows; ++i) nn += dst[i] * dst[i];
        if (nn > 0.5) continue;
        for (std::size_t cand = 0; cand < rows; ++cand) {
            std::fill(dst, dst + rows, 0.0);
            dst[cand] = 1.0;
            for (int pass = 0; pass < 2; ++pass)
                for (std::size_t o = 0; o < cols; ++o) {
                    if (o == jj) continue;
                    const double* other = ud.data() + o * rows;
                    double dt = 0;
                    for (std::size_t i = 0; i < rows; ++i) dt += other[i] * dst[i];
                    for (std::size_t i = 0; i < rows; ++i) dst[i] -= dt * other[i];
                }
            double n2 = 0;
            for (std::size_t i = 0; i < rows; ++i) n2 += dst[i] * dst[i];
            if (n2 > 0.25) {
                const double inv = 1.0 / std::sqrt(n2);
                for (std::size_t i = 0; i < rows; ++i) dst[i] *= inv;
                break;
            }
        }
    }
    u.resize(rows * cols);
    for (std::size_t k = 0; k < u.size(); ++k) u[k] = static_cast<T>(ud[k]);
}
template void thin_svd(const float*, std::size_t, std::size_t, std::vector<float>&, std::vector<float>&);
template void thin_svd(const double*, std::size_t, std::size_t, std::vector<double>&, std::vector<double>&);

}  // namespace orc
