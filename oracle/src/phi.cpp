// ORACLE (test infrastructure): phi functions and the adaptive Krylov engine.
// Restates proj/src/phi.cpp; expm restates the published Higham (2005)
// scaling-and-squaring algorithm that Eigen's MatrixFunctions implements.
#include <algorithm>
#include <cmath>

#include "oracle.hpp"

namespace oracle {

namespace {
double factorial(int i) {
  double f = 1.0;
  for (int j = 2; j <= i; ++j) f *= j;
  return f;
}

// LU with partial pivoting, solves A X = B in place (B overwritten by X).
void lu_solve(Mat a, Mat& b) {
  const int n = a.r;
  std::vector<int> piv(n);
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(a(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a(i, k)) > best) { best = std::abs(a(i, k)); p = i; }
    piv[k] = p;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(a(k, j), a(p, j));
      for (int j = 0; j < b.c; ++j) std::swap(b(k, j), b(p, j));
    }
    const double d = a(k, k);
    for (int i = k + 1; i < n; ++i) {
      const double l = a(i, k) / d;
      a(i, k) = l;
      for (int j = k + 1; j < n; ++j) a(i, j) -= l * a(k, j);
      for (int j = 0; j < b.c; ++j) b(i, j) -= l * b(k, j);
    }
  }
  for (int j = 0; j < b.c; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = b(i, j);
      for (int k = i + 1; k < n; ++k) s -= a(i, k) * b(k, j);
      b(i, j) = s / a(i, i);
    }
}

Mat lincomb(std::initializer_list<std::pair<double, const Mat*>> terms, double ident) {
  const Mat& first = *terms.begin()->second;
  Mat out(first.r, first.c);
  for (auto& [c, m] : terms)
    for (size_t i = 0; i < out.a.size(); ++i) out.a[i] += c * m->a[i];
  for (int i = 0; i < out.r; ++i) out(i, i) += ident;
  return out;
}
}  // namespace

// proj/src/phi.cpp:19-38
double phi_scalar(int i, double tau) {
  if (i < 0 || i > 6) throw std::invalid_argument("phi_scalar: i must be in [0, 6]");
  if (i == 0) return std::exp(tau);
  if (std::abs(tau) < 4.0) {
    double term = 1.0 / factorial(i);
    double sum = term;
    for (int j = 1; j < 60; ++j) {
      term *= tau / (i + j);
      sum += term;
      if (std::abs(term) < 1e-18 * std::abs(sum)) break;
    }
    return sum;
  }
  double phi = std::exp(tau);
  for (int k = 0; k < i; ++k) phi = (phi - 1.0 / factorial(k)) / tau;
  return phi;
}

// proj/src/phi.cpp:40 (Eigen MatrixFunctions exp): Higham 2005, "The scaling
// and squaring method for the matrix exponential revisited", Algorithm 2.3 —
// diagonal Pade degree 3/5/7/9 chosen by the 1-norm against theta_m, else
// degree 13 after scaling by 2^-s with s from frexp(||A||_1 / theta_13).
Mat expm(const Mat& m) {
  const int n = m.r;
  double l1 = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::abs(m(i, j));
    l1 = std::max(l1, s);
  }
  Mat U, V;
  int squarings = 0;
  Mat A = m;
  if (l1 < 1.495585217958292e-002) {
    static const double b[] = {120.0, 60.0, 12.0, 1.0};
    const Mat A2 = matmul(A, A);
    const Mat tmp = lincomb({{b[3], &A2}}, b[1]);
    U = matmul(A, tmp);
    V = lincomb({{b[2], &A2}}, b[0]);
  } else if (l1 < 2.539398330063230e-001) {
    static const double b[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
    const Mat A2 = matmul(A, A), A4 = matmul(A2, A2);
    const Mat tmp = lincomb({{b[5], &A4}, {b[3], &A2}}, b[1]);
    U = matmul(A, tmp);
    V = lincomb({{b[4], &A4}, {b[2], &A2}}, b[0]);
  } else if (l1 < 9.504178996162932e-001) {
    static const double b[] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
    const Mat A2 = matmul(A, A), A4 = matmul(A2, A2), A6 = matmul(A4, A2);
    const Mat tmp = lincomb({{b[7], &A6}, {b[5], &A4}, {b[3], &A2}}, b[1]);
    U = matmul(A, tmp);
    V = lincomb({{b[6], &A6}, {b[4], &A4}, {b[2], &A2}}, b[0]);
  } else if (l1 < 2.097847961257068e+000) {
    static const double b[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                               2162160.0,     110880.0,     3960.0,       90.0,        1.0};
    const Mat A2 = matmul(A, A), A4 = matmul(A2, A2), A6 = matmul(A4, A2), A8 = matmul(A6, A2);
    const Mat tmp = lincomb({{b[9], &A8}, {b[7], &A6}, {b[5], &A4}, {b[3], &A2}}, b[1]);
    U = matmul(A, tmp);
    V = lincomb({{b[8], &A8}, {b[6], &A6}, {b[4], &A4}, {b[2], &A2}}, b[0]);
  } else {
    static const double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                               1187353796428800.0,  129060195264000.0,   10559470521600.0,
                               670442572800.0,      33522128640.0,       1323241920.0,
                               40840800.0,          960960.0,            16380.0,
                               182.0,               1.0};
    const double maxnorm = 5.371920351148152;
    std::frexp(l1 / maxnorm, &squarings);
    if (squarings < 0) squarings = 0;
    for (auto& x : A.a) x = std::ldexp(x, -squarings);
    const Mat A2 = matmul(A, A), A4 = matmul(A2, A2), A6 = matmul(A4, A2);
    const Mat t1 = lincomb({{b[13], &A6}, {b[11], &A4}, {b[9], &A2}}, 0.0);
    Mat t2 = matmul(A6, t1);
    const Mat tmp = lincomb({{1.0, &t2}, {b[7], &A6}, {b[5], &A4}, {b[3], &A2}}, b[1]);
    U = matmul(A, tmp);
    const Mat t3 = lincomb({{b[12], &A6}, {b[10], &A4}, {b[8], &A2}}, 0.0);
    const Mat t4 = matmul(A6, t3);
    V = lincomb({{1.0, &t4}, {b[6], &A6}, {b[4], &A4}, {b[2], &A2}}, b[0]);
  }
  Mat numer = lincomb({{1.0, &U}, {1.0, &V}}, 0.0);
  const Mat denom = lincomb({{-1.0, &U}, {1.0, &V}}, 0.0);
  lu_solve(denom, numer);
  for (int i = 0; i < squarings; ++i) numer = matmul(numer, numer);
  return numer;
}

// proj/src/phi.cpp:42-56
std::vector<Mat> phi_dense_family(int p, const Mat& m) {
  const int n = m.r;
  if (m.c != n) throw std::invalid_argument("phi_dense: square matrix required");
  if (p == 0) return {expm(m)};
  const int big = (p + 1) * n;
  Mat block(big, big);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) block(i, j) = m(i, j);
  for (int j = 0; j < p; ++j)
    for (int i = 0; i < n; ++i) block(j * n + i, (j + 1) * n + i) = 1.0;
  const Mat e = expm(block);
  std::vector<Mat> fam;
  for (int j = 0; j <= p; ++j) {
    Mat f(n, n);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < n; ++c) f(r, c) = e(r, j * n + c);
    fam.push_back(f);
  }
  return fam;
}

// proj/src/phi.cpp:58-61
Mat phi_dense(int i, const Mat& m) {
  if (i < 0 || i > 6) throw std::invalid_argument("phi_dense: i must be in [0, 6]");
  return phi_dense_family(i, m).back();
}

namespace {
// proj/src/phi.cpp:66-113 — incrementally extendable Arnoldi / IOP workspace,
// modified Gram-Schmidt with two passes under full orthogonalization.
struct ArnoldiWorkspace {
  std::vector<Vec> V;
  Mat H;
  int m = 0;
  double beta = 0;
  bool breakdown = false;

  void reset(const Vec& seed, int mmax) {
    V.assign(mmax + 1, Vec());
    H = Mat(mmax + 1, mmax);
    beta = norm(seed);
    V[0] = Vec(seed.size());
    for (size_t i = 0; i < seed.size(); ++i) V[0][i] = seed[i] / beta;
    m = 0;
    breakdown = false;
  }

  long extend(const LinearAction& op, int target, int window) {
    long applies = 0;
    const int mmax = H.c;
    while (m < target && !breakdown) {
      Vec w = op(V[m]);
      ++applies;
      const double pre_norm = norm(w);
      const bool full = window >= mmax;
      const int j0 = full ? 0 : std::max(0, m + 1 - window);
      const int passes = full ? 2 : 1;
      for (int pass = 0; pass < passes; ++pass)
        for (int j = j0; j <= m; ++j) {
          const double hjm = dot(V[j], w);
          for (size_t i = 0; i < w.size(); ++i) w[i] -= hjm * V[j][i];
          H(j, m) += hjm;
        }
      const double hnext = norm(w);
      H(m + 1, m) = hnext;
      ++m;
      if (hnext <= 1e-14 * std::max(pre_norm, 1e-300)) {
        H(m, m - 1) = 0.0;
        breakdown = true;
        break;
      }
      V[m] = Vec(w.size());
      for (size_t i = 0; i < w.size(); ++i) V[m][i] = w[i] / hnext;
    }
    return applies;
  }
};
}  // namespace

// proj/src/phi.cpp:117-131
KrylovFactorization krylov_build(const LinearAction& op, const Vec& seed, int m, int orth_length) {
  if (norm(seed) == 0.0) throw std::invalid_argument("krylov_build: zero seed");
  ArnoldiWorkspace ws;
  ws.reset(seed, m);
  ws.extend(op, m, orth_length >= m ? m : orth_length);
  KrylovFactorization f;
  f.m = ws.m;
  f.seed_norm = ws.beta;
  f.invariant_subspace = ws.breakdown;
  const int cols = ws.m + (ws.breakdown ? 0 : 1);
  const int n = int(seed.size());
  f.basis = Mat(n, cols);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < n; ++i) f.basis(i, j) = ws.V[j][i];
  f.hessenberg = Mat(ws.m + 1, ws.m);
  for (int i = 0; i <= ws.m; ++i)
    for (int j = 0; j < ws.m; ++j) f.hessenberg(i, j) = ws.H(i, j);
  return f;
}

// proj/src/phi.cpp:133-260 — adaptive augmented-Krylov phi combination.
PhiCombinationResult phi_combination(const PhiCombinationProblem& prob) {
  if (prob.b.empty()) throw std::invalid_argument("phi_combination: empty b list");
  if (!(prob.dt > 0.0)) throw std::invalid_argument("phi_combination: dt must be positive");
  const long n = long(prob.b.front().size());
  const int p = int(prob.b.size()) - 1;
  for (const auto& bi : prob.b)
    if (long(bi.size()) != n) throw std::invalid_argument("phi_combination: inconsistent sizes");
  PhiCombinationResult res;
  res.value.assign(n, 0.0);
  bool any = false;
  for (const auto& bi : prob.b) any = any || norm(bi) > 0.0;
  if (!any) return res;

  const long dim = n + p;
  const double dt = prob.dt;
  auto aug_op = [&](const Vec& x) {
    Vec y(dim);
    const Vec head(x.begin(), x.begin() + n);
    const Vec lh = prob.op(head);
    for (long i = 0; i < n; ++i) y[i] = lh[i];
    for (int j = 0; j < p; ++j)
      for (long i = 0; i < n; ++i) y[i] += x[n + j] * prob.b[p - j][i];
    for (int j = 0; j + 1 < p; ++j) y[n + j] = x[n + j + 1];
    if (p > 0) y[n + p - 1] = 0.0;
    for (auto& v : y) v = dt * v;
    return y;
  };

  Vec w(dim, 0.0);
  for (long i = 0; i < n; ++i) w[i] = prob.b[0][i];
  if (p > 0) w[dim - 1] = 1.0;

  const double tol = std::max(prob.tol, 5e-15);
  const int mmax = int(std::min<long>(prob.max_basis, dim));
  const bool full_orth = prob.orth_length >= mmax || dim <= std::max(prob.initial_basis, 16);
  const int window = full_orth ? mmax : prob.orth_length;
  const int grow_cap = full_orth ? mmax : std::min(mmax, 32);

  ArnoldiWorkspace ws;
  double t = 0.0, h = 1.0;
  int m = std::min(prob.initial_basis, mmax);
  double last_estimate = 0.0;

  while (t < 1.0 - 1e-14) {
    if (res.stats.substeps >= prob.max_substeps)
      throw KrylovError("phi_combination: no convergence within substep budget", last_estimate);
    const double beta = norm(w);
    if (beta == 0.0) break;
    if (!std::isfinite(beta)) throw KrylovError("phi_combination: non-finite input", beta);
    ws.reset(w, mmax);
    res.stats.iterations += ws.extend(aug_op, m, window);
    double avnorm = 0.0;
    if (!ws.breakdown) {
      avnorm = norm(aug_op(ws.V[ws.m]));
      ++res.stats.iterations;
    }
    bool accepted = false;
    while (!accepted) {
      const int mc = ws.m;
      Mat hbar(mc + 2, mc + 2);
      for (int i = 0; i <= mc; ++i)
        for (int j = 0; j < mc; ++j) hbar(i, j) = ws.H(i, j);
      hbar(mc + 1, mc) = 1.0;
      Mat hh = hbar;
      for (auto& x : hh.a) x = h * x;
      const Mat f = expm(hh);
      double err_loc = 0.0;
      if (!ws.breakdown) {
        const double p1 = std::abs(beta * f(mc, 0));
        const double p2 = std::abs(beta * f(mc + 1, 0)) * avnorm;
        if (p1 > 10.0 * p2) err_loc = p2;
        else if (p1 > p2) err_loc = p1 * p2 / (p1 - p2);
        else err_loc = p1;
      }
      last_estimate = err_loc;
      if (ws.breakdown || err_loc <= 0.5 * tol * beta * h) {
        // w = V(:, 0:mc) * (beta * f(0:mc, 0))
        Vec coef(mc);
        for (int j = 0; j < mc; ++j) coef[j] = beta * f(j, 0);
        Vec nw(dim, 0.0);
        for (long i = 0; i < dim; ++i) {
          double s = 0.0;
          for (int j = 0; j < mc; ++j) s += ws.V[j][i] * coef[j];
          nw[i] = s;
        }
        w = nw;
        t += h;
        ++res.stats.substeps;
        for (int j = 0; j < p; ++j) {
          double v = 1.0;
          for (int q = 1; q <= p - 1 - j; ++q) v *= dt * t / q;
          w[n + j] = v;
        }
        accepted = true;
        if (err_loc < 1e-3 * tol * beta * h) h *= 2.0;
        h = std::min(h, 1.0 - t);
      } else if (mc < grow_cap) {
        m = std::min(grow_cap, std::max(mc + 1, (3 * mc) / 2));
        res.stats.iterations += ws.extend(aug_op, m, window);
        if (!ws.breakdown) {
          avnorm = norm(aug_op(ws.V[ws.m]));
          ++res.stats.iterations;
        }
      } else {
        h *= 0.5;
        if (h < 1e-12) throw KrylovError("phi_combination: substep underflow", err_loc);
      }
    }
  }
  res.value.assign(w.begin(), w.begin() + n);
  return res;
}

}  // namespace oracle
