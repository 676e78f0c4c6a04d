// plan.cpp — host planner for joint-cut HSF (arXiv 2502.06959).
//
// Steps (all fp64, host, once per plan — off the timed path):
//   H1 parse + validate the circuit file                     (DESIGN.md format)
//   H2 classify, contract blocks in the wire DAG, Kahn schedule;
//      non-convex block => HSF_ERR_NONCONVEX_BLOCK
//   H3 block assembly: dense product of embedded members, or the diagonal
//      route when every member is diagonal
//   H4 reshape / matricise  A~[(i^b,j^b),(i^a,j^a)]         (Eq. 5-6)
//   H5 one-sided complex Jacobi SVD                          (Eq. 7)
//   H6 truncate sigma_m <= tol*sigma_0; absorb U, V* into Y_m, X_m (Eq. 8-9,
//      P:177-181); rescale to unitary-scale factors
//   H7 radices, n_p = prod r_u, path budget
//   H8 per-half programs: fixed local gates + factor slots, gate fusion
//      (P:282), path-tree levels, SMEM tile passes
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <array>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <queue>
#include <set>
#include <sstream>

#include "hsf_internal.h"

namespace hsf {

[[noreturn]] void fail(hsf_status st, const std::string& msg) { throw Error{st, msg}; }

// ------------------------------------------------------------- gate library
static std::vector<cd> diag_mat(std::initializer_list<cd> d) {
  int n = (int)d.size();
  std::vector<cd> U(n * n, 0.0);
  int i = 0;
  for (cd v : d) { U[i * n + i] = v; ++i; }
  return U;
}

static Gate make_named(const std::string& name, const std::vector<double>& prm, const std::vector<int>& q) {
  Gate g;
  g.name = name;
  g.q = q;
  g.k = (int)q.size();
  const double s2 = 1.0 / std::sqrt(2.0);
  const cd I(0, 1);
  if (name == "h") g.U = {s2, s2, s2, -s2};
  else if (name == "x") g.U = {0.0, 1.0, 1.0, 0.0};
  else if (name == "z") g.U = diag_mat({1.0, -1.0});
  else if (name == "rx") {
    double c = std::cos(prm[0] / 2), s = std::sin(prm[0] / 2);
    g.U = {c, -I * s, -I * s, c};
  } else if (name == "rz") g.U = diag_mat({std::exp(-I * (prm[0] / 2)), std::exp(I * (prm[0] / 2))});
  else if (name == "cz") g.U = diag_mat({1.0, 1.0, 1.0, -1.0});
  else if (name == "cx") {  // control = first listed (MSB): P0 (x) I + P1 (x) X
    g.U.assign(16, 0.0);
    g.U[0 * 4 + 0] = 1; g.U[1 * 4 + 1] = 1; g.U[2 * 4 + 3] = 1; g.U[3 * 4 + 2] = 1;
  } else if (name == "swap") {
    g.U.assign(16, 0.0);
    g.U[0] = 1; g.U[1 * 4 + 2] = 1; g.U[2 * 4 + 1] = 1; g.U[15] = 1;
  } else if (name == "cp") g.U = diag_mat({1.0, 1.0, 1.0, std::exp(I * prm[0])});
  else if (name == "rzz") {
    cd a = std::exp(-I * (prm[0] / 2)), b = std::exp(I * (prm[0] / 2));
    g.U = diag_mat({a, b, b, a});
  } else fail(HSF_ERR_UNSUPPORTED_GATE, "unsupported gate '" + name + "'");
  return g;
}

static bool is_diag(const Gate& g) {
  int d = 1 << g.k;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (i != j && g.U[i * d + j] != cd(0.0)) return false;
  return true;
}

// --------------------------------------------------------------- H1 parser
static std::vector<Gate> parse(const char* text, size_t len, int* n_out) {
  std::string s(text, len);
  std::istringstream in(s);
  std::string line;
  int n = -1, lineno = 0;
  std::vector<Gate> gates;
  static const std::map<std::string, std::pair<int, int>> arity = {
      {"h", {0, 1}}, {"x", {0, 1}}, {"z", {0, 1}}, {"rx", {1, 1}}, {"rz", {1, 1}},
      {"cz", {0, 2}}, {"cx", {0, 2}}, {"swap", {0, 2}}, {"cp", {1, 2}}, {"rzz", {1, 2}}};
  auto num = [&](const std::string& t) {
    char* e = nullptr;
    double v = std::strtod(t.c_str(), &e);
    if (e == t.c_str() || *e) fail(HSF_ERR_PARSE, "line " + std::to_string(lineno) + ": bad number '" + t + "'");
    return v;
  };
  auto integer = [&](const std::string& t) {
    char* e = nullptr;
    long v = std::strtol(t.c_str(), &e, 10);
    if (e == t.c_str() || *e) fail(HSF_ERR_PARSE, "line " + std::to_string(lineno) + ": bad integer '" + t + "'");
    return (int)v;
  };
  while (std::getline(in, line)) {
    ++lineno;
    auto h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    std::string t;
    while (ls >> t) tok.push_back(t);
    if (tok.empty()) continue;
    if (tok[0] == "qubits") {
      if (tok.size() != 2) fail(HSF_ERR_PARSE, "line " + std::to_string(lineno) + ": 'qubits <n>'");
      n = integer(tok[1]);
      if (n < 2 || n > 64) fail(HSF_ERR_INVALID_ARG, "qubits must be in [2,64]");
      continue;
    }
    if (n < 0) fail(HSF_ERR_PARSE, "line " + std::to_string(lineno) + ": gate before 'qubits'");
    Gate g;
    if (tok[0] == "u") {
      if (tok.size() < 2) fail(HSF_ERR_PARSE, "line " + std::to_string(lineno) + ": 'u k q.. reals'");
      int k = integer(tok[1]);
      if (k < 1 || k > 12) fail(HSF_ERR_UNSUPPORTED_GATE, "u gate arity must be 1..12");
      size_t need = 2 + (size_t)k + 2 * ((size_t)1 << (2 * k));
      if (tok.size() != need) fail(HSF_ERR_PARSE, "line " + std::to_string(lineno) + ": bad u payload length");
      g.name = "u";
      g.k = k;
      for (int j = 0; j < k; ++j) g.q.push_back(integer(tok[2 + j]));
      size_t d2 = (size_t)1 << (2 * k);
      g.U.resize(d2);
      for (size_t e = 0; e < d2; ++e) g.U[e] = cd(num(tok[2 + k + 2 * e]), num(tok[3 + k + 2 * e]));
    } else {
      auto it = arity.find(tok[0]);
      if (it == arity.end()) fail(HSF_ERR_UNSUPPORTED_GATE, "line " + std::to_string(lineno) + ": unknown gate '" + tok[0] + "'");
      int np = it->second.first, nq = it->second.second;
      if ((int)tok.size() != 1 + np + nq) fail(HSF_ERR_UNSUPPORTED_GATE, "line " + std::to_string(lineno) + ": wrong arity");
      std::vector<double> prm;
      std::vector<int> q;
      for (int j = 0; j < np; ++j) prm.push_back(num(tok[1 + j]));
      for (int j = 0; j < nq; ++j) q.push_back(integer(tok[1 + np + j]));
      g = make_named(tok[0], prm, q);
    }
    std::set<int> seen;
    for (int q : g.q) {
      if (q < 0 || q >= n) fail(HSF_ERR_DUPLICATE_QUBIT, "line " + std::to_string(lineno) + ": qubit out of range");
      if (!seen.insert(q).second) fail(HSF_ERR_DUPLICATE_QUBIT, "line " + std::to_string(lineno) + ": duplicate qubit");
    }
    g.diag = is_diag(g);
    gates.push_back(std::move(g));
  }
  if (n < 0) fail(HSF_ERR_PARSE, "missing 'qubits' line");
  *n_out = n;
  return gates;
}

// ------------------------------------------------------------- linear algebra
// Embed gate g into a block-local space whose bit t is support[t].
static std::vector<cd> embed(const Gate& g, const std::vector<int>& support) {
  const int ks = (int)support.size();
  const size_t N = (size_t)1 << ks;
  std::vector<int> pos(g.k);
  for (int j = 0; j < g.k; ++j)
    pos[j] = (int)(std::find(support.begin(), support.end(), g.q[j]) - support.begin());
  std::vector<cd> E(N * N, 0.0);
  const int dg = 1 << g.k;
  for (size_t col = 0; col < N; ++col) {
    int jl = 0;
    for (int j = 0; j < g.k; ++j) jl = (jl << 1) | (int)((col >> pos[j]) & 1);
    size_t clear = col;
    for (int j = 0; j < g.k; ++j) clear &= ~((size_t)1 << pos[j]);
    for (int il = 0; il < dg; ++il) {
      size_t row = clear;
      for (int j = 0; j < g.k; ++j) row |= (size_t)((il >> (g.k - 1 - j)) & 1) << pos[j];
      E[row * N + col] += g.U[(size_t)il * dg + jl];
    }
  }
  return E;
}

static std::vector<cd> matmul(const std::vector<cd>& A, const std::vector<cd>& B, size_t N) {
  std::vector<cd> C(N * N, 0.0);
  for (size_t i = 0; i < N; ++i)
    for (size_t k = 0; k < N; ++k) {
      cd a = A[i * N + k];
      if (a == cd(0.0)) continue;
      for (size_t j = 0; j < N; ++j) C[i * N + j] += a * B[k * N + j];
    }
  return C;
}

// One-sided (Hestenes) complex Jacobi SVD of an R x C matrix (row-major).
// Returns sigma (descending), U (R x r, column m = left vector), V (C x r).
struct Svd {
  std::vector<double> s;
  std::vector<std::vector<cd>> u, v;  // per singular triple
};

static Svd jacobi_svd_tall(const std::vector<cd>& M, int R, int C) {
  // columns of A (R x C) as separate vectors
  std::vector<std::vector<cd>> a(C, std::vector<cd>(R)), v(C, std::vector<cd>(C, 0.0));
  for (int j = 0; j < C; ++j) {
    for (int i = 0; i < R; ++i) a[j][i] = M[(size_t)i * C + j];
    v[j][j] = 1.0;
  }
  // convergence: |a_i^H a_j| <= tol * |a_i||a_j|, plus an absolute floor so
  // pairs of round-off-level columns (zero singular values) do not rotate forever
  const double tol = 1e-15 * std::max(1.0, std::sqrt((double)R));
  double frob2 = 0;
  for (const cd& x : M) frob2 += std::norm(x);
  const double floor_abs = 1e-32 * frob2;
  bool converged = false;
  for (int sweep = 0; sweep < 80 && !converged; ++sweep) {
    converged = true;
    for (int i = 0; i < C - 1; ++i)
      for (int j = i + 1; j < C; ++j) {
        double al = 0, be = 0;
        cd ga = 0;
        for (int r = 0; r < R; ++r) {
          al += std::norm(a[i][r]);
          be += std::norm(a[j][r]);
          ga += std::conj(a[i][r]) * a[j][r];
        }
        double g = std::abs(ga);
        if (g <= floor_abs || g <= tol * std::sqrt(al * be)) continue;
        converged = false;
        cd ph = ga / g;  // e^{i phi}
        double zeta = (be - al) / (2.0 * g);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        cd sph = s * std::conj(ph), cph = c * std::conj(ph);
        for (int r = 0; r < R; ++r) {
          cd x = a[i][r], y = a[j][r];
          a[i][r] = c * x - sph * y;
          a[j][r] = s * x + cph * y;
        }
        for (int r = 0; r < C; ++r) {
          cd x = v[i][r], y = v[j][r];
          v[i][r] = c * x - sph * y;
          v[j][r] = s * x + cph * y;
        }
      }
  }
  if (!converged) fail(HSF_ERR_SVD_NO_CONVERGENCE, "Jacobi SVD did not converge in 80 sweeps");
  std::vector<int> idx(C);
  std::vector<double> nrm(C);
  for (int j = 0; j < C; ++j) {
    double s = 0;
    for (int r = 0; r < R; ++r) s += std::norm(a[j][r]);
    nrm[j] = std::sqrt(s);
    idx[j] = j;
  }
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
  Svd out;
  for (int j : idx) {
    out.s.push_back(nrm[j]);
    std::vector<cd> u(R);
    for (int r = 0; r < R; ++r) u[r] = nrm[j] > 0 ? a[j][r] / nrm[j] : cd(0.0);
    out.u.push_back(std::move(u));
    out.v.push_back(v[j]);
  }
  return out;
}

static Svd jacobi_svd(const std::vector<cd>& M, int R, int C) {
  if (C <= R) return jacobi_svd_tall(M, R, C);
  // M^H = U' S V'^H  =>  M = V' S U'^H
  std::vector<cd> MH((size_t)C * R);
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < C; ++j) MH[(size_t)j * R + i] = std::conj(M[(size_t)i * C + j]);
  Svd t = jacobi_svd_tall(MH, C, R);
  std::swap(t.u, t.v);
  return t;
}

// ----------------------------------------------------- H3-H6 one cut unit
// Analytic cascade route (Eq. 11; "analytical expressions
// can be found for cascade structures"): every member is a two-qubit gate on
// one common qubit c and block-diagonal in c's computational basis,
// G = P0_c (x) G_0 + P1_c (x) G_1 (CNOT: G_0 = I, G_1 = X; CZ, CP, RZZ: diagonal
// G_v).  Members on distinct targets commute inside each c-sector, so
//   U_S = sum_{v=0,1} P_v,c (x) prod_t G_{t,v}
//       = O_0 (x) N_0 + O_1 (x) N_1,
// O_v on c's side (P_v (x) that side's targets' products, Frobenius-orthogonal
// with equal norms alpha), N_v on the other side (unitary, norm beta).  The
// reshaped matrix (Eq. 6) then has rank <= 2 and its SVD is closed-form: the
// 2 x 2 Gram matrix of the N_v, [[beta, g], [conj g, beta]] with
// g = <N_0, N_1>_F, has eigenvalues beta +- |g| and eigenvectors
// (1, +-conj(g)/|g|) / sqrt 2, so sigma_+- = sqrt(alpha (beta +- |g|)) and the
// Schmidt pairs are the Gram-rotated combinations (Eq. 7-9) -- no block
// assembly, no iterative SVD.  Returns false (numeric route) when the block
// is not such a cascade.  (For degenerate sigma -- g = 0, e.g. CNOT cascades --
// the factors are one valid basis of the degenerate pair; the path sum over
// all terms is the same for every basis, partial sums of a degenerate pair's
// terms are not unique, SURVEY §8(c) reading 6.)
static bool analytic_cascade(const std::vector<Gate>& gates, Unit& u, int n_low, const hsf_plan_opts& o) {
  // cascades of >= 2 gates; a single crossing gate keeps the numeric route
  // (its SVD is tiny, and it then shares LAPACK's basis for degenerate sigma)
  if (u.gids.size() < 2) return false;
  std::set<int> common;
  for (size_t i = 0; i < u.gids.size(); ++i) {
    const Gate& g = gates[u.gids[i]];
    if (g.k != 2) return false;
    std::set<int> qs(g.q.begin(), g.q.end());
    if (i == 0) {
      common = qs;
    } else {
      std::set<int> inter;
      for (int q : qs)
        if (common.count(q)) inter.insert(q);
      common.swap(inter);
    }
  }
  for (int c : common) {
    // G_v of every member as a 2 x 2 matrix on its target, block-diagonality checked
    std::vector<std::array<std::array<cd, 4>, 2>> Gv(u.gids.size());
    std::vector<int> tgt(u.gids.size());
    bool ok = true;
    for (size_t i = 0; i < u.gids.size() && ok; ++i) {
      const Gate& g = gates[u.gids[i]];
      const bool cmsb = g.q[0] == c;  // first-listed qubit = MSB of the gate-local index
      tgt[i] = cmsb ? g.q[1] : g.q[0];
      auto idx = [&](int v, int t) { return cmsb ? (v << 1) | t : (t << 1) | v; };
      for (int vi = 0; vi < 2 && ok; ++vi)
        for (int ti = 0; ti < 2; ++ti)
          for (int vj = 0; vj < 2; ++vj)
            for (int tj = 0; tj < 2; ++tj) {
              const cd x = g.U[(size_t)idx(vi, ti) * 4 + idx(vj, tj)];
              if (vi != vj) {
                if (x != cd(0.0)) ok = false;
              } else {
                Gv[i][vi][ti * 2 + tj] = x;
              }
            }
    }
    if (!ok) continue;
    const bool diag = u.diag_route;
    const bool c_low = c < n_low;
    const std::vector<int>& So = c_low ? u.Sb : u.Sa;  // c's side
    const std::vector<int>& Sn = c_low ? u.Sa : u.Sb;  // the other side
    const int ko = (int)So.size(), kn = (int)Sn.size();
    if (!diag && (ko > 5 || kn > 5)) return false;  // dense factors of <= 5 qubits per half (device limit)
    // per-qubit 2 x 2 products (later gates on the left), per sector v
    auto side_op = [&](const std::vector<int>& S, int v, bool with_proj) {
      const size_t d = (size_t)1 << S.size();
      std::vector<std::array<cd, 4>> per(S.size());
      for (size_t j = 0; j < S.size(); ++j) per[j] = {1.0, 0.0, 0.0, 1.0};
      for (size_t i = 0; i < u.gids.size(); ++i) {
        const size_t j = (size_t)(std::find(S.begin(), S.end(), tgt[i]) - S.begin());
        if (j == S.size()) continue;
        const auto& G = Gv[i][v];
        const auto P = per[j];
        per[j] = {G[0] * P[0] + G[1] * P[2], G[0] * P[1] + G[1] * P[3], G[2] * P[0] + G[3] * P[2],
                  G[2] * P[1] + G[3] * P[3]};
      }
      if (with_proj) {
        const size_t jc = (size_t)(std::find(S.begin(), S.end(), c) - S.begin());
        per[jc] = v == 0 ? std::array<cd, 4>{1.0, 0.0, 0.0, 0.0} : std::array<cd, 4>{0.0, 0.0, 0.0, 1.0};
      }
      // tensor product, local index LSB = smallest support qubit (S ascending)
      std::vector<cd> M(diag ? d : d * d);
      for (size_t r = 0; r < d; ++r)
        for (size_t col = 0; col < (diag ? 1 : d); ++col) {
          const size_t cc = diag ? r : col;
          cd x = 1.0;
          for (size_t j = 0; j < S.size(); ++j) x *= per[j][((r >> j) & 1) * 2 + ((cc >> j) & 1)];
          M[diag ? r : r * d + col] = x;
        }
      return M;
    };
    std::vector<cd> O0 = side_op(So, 0, true), O1 = side_op(So, 1, true);
    std::vector<cd> N0 = side_op(Sn, 0, false), N1 = side_op(Sn, 1, false);
    auto inner = [](const std::vector<cd>& A, const std::vector<cd>& B) {
      cd s = 0.0;
      for (size_t e = 0; e < A.size(); ++e) s += std::conj(A[e]) * B[e];
      return s;
    };
    const double alpha = std::real(inner(O0, O0)), beta = std::real(inner(N0, N0));
    const cd g = inner(N0, N1);
    const double ag = std::abs(g);
    const cd ph = ag > 0 ? std::conj(g) / ag : cd(1.0);
    // M = [u_+, u_-] (columns), u_+- = (1, +-ph) / sqrt 2; |g| = 0: identity
    cd M[2][2];
    if (ag > 0) {
      const double r2 = 1.0 / std::sqrt(2.0);
      M[0][0] = r2, M[1][0] = ph * r2, M[0][1] = r2, M[1][1] = -ph * r2;
    } else {
      M[0][0] = 1.0, M[1][0] = 0.0, M[0][1] = 0.0, M[1][1] = 1.0;
    }
    // lambda_k = || sum_v M_vk N_v ||^2 (= beta +- |g|), from the combined vectors:
    // the difference form keeps the small sigma accurate (no beta - |g| cancellation)
    std::vector<cd> Nc[2];
    double lam[2];
    for (int k = 0; k < 2; ++k) {
      Nc[k].resize(N0.size());
      for (size_t e = 0; e < N0.size(); ++e) Nc[k][e] = M[0][k] * N0[e] + M[1][k] * N1[e];
      lam[k] = std::real(inner(Nc[k], Nc[k]));
    }
    const double s0 = std::sqrt(alpha * lam[0]);
    const int na = (int)u.Sa.size(), nb = (int)u.Sb.size();
    const double sa = std::sqrt((double)(1 << na)), sb = std::sqrt((double)(1 << nb));
    for (int k = 0; k < 2; ++k) {
      const double sig = std::sqrt(std::max(0.0, alpha * lam[k]));
      if (!(sig > o.svd_rel_tol * s0)) break;
      // N^_k = sum_v M_vk N_v (unit norm / sqrt(lam)), O^_k = sum_w conj(M_wk) O_w (/ sqrt(alpha))
      std::vector<cd> Nk(N0.size()), Ok(O0.size());
      for (size_t e = 0; e < Nk.size(); ++e) Nk[e] = Nc[k][e] / std::sqrt(lam[k]);
      for (size_t e = 0; e < Ok.size(); ++e)
        Ok[e] = (std::conj(M[0][k]) * O0[e] + std::conj(M[1][k]) * O1[e]) / std::sqrt(alpha);
      std::vector<cd>& xa = c_low ? Nk : Ok;  // side a (high)
      std::vector<cd>& yb = c_low ? Ok : Nk;  // side b (low)
      for (auto& x : xa) x *= sa;  // unitary-scale factors, c = sigma / sqrt(2^|S|) (reading 4)
      for (auto& y : yb) y *= sb;
      u.sigma.push_back(sig);
      u.c.push_back(cd(sig / (sa * sb), 0.0));
      u.X.push_back(std::move(xa));
      u.Y.push_back(std::move(yb));
    }
    u.rank = (int)u.sigma.size();
    u.analytic = true;
    return true;
  }
  return false;
}

// Sequential (MPO-style) route for dense blocks (assembly and SVD
// of a block cost O(D^s + D^3); "keep blocks small"): the block operator is
// carried as a sum of terms X_k (x) Y_k over its two sides and built gate by
// gate in application order -- a gate inside one side multiplies that side's
// factors, a crossing gate G = sum_j g^a_j (x) g^b_j (its own operator-Schmidt
// decomposition, Eq. 6-9 on the gate) multiplies every term by every pair --
// and after each crossing gate the terms are recompressed to the operator
// Schmidt form: orthonormal bases of span{X_k} and span{Y_k} (SVDs of the
// stacked factors), the small coefficient matrix C_ij = <x^_i (x) y^_j, U>
// and its SVD.  The result is the SVD of the reshaped block (Eq. 6) without
// forming the 2^s x 2^s block matrix or the 4^s_b x 4^s_a reshaped one: for a
// 5 + 5 brickwork block, milliseconds instead of seconds.  sigma and the
// factors equal the dense route's up to the basis of degenerate sigma (the
// path sum over all terms is basis-independent, SURVEY reading 6).
static void sequential_unit(const std::vector<Gate>& gates, Unit& u, const hsf_plan_opts& o) {
  const int na = (int)u.Sa.size(), nb = (int)u.Sb.size();
  const size_t da = (size_t)1 << na, db = (size_t)1 << nb, ea = da * da, eb = db * db;
  std::vector<std::vector<cd>> X(1, std::vector<cd>(ea, 0.0)), Y(1, std::vector<cd>(eb, 0.0));
  for (size_t i = 0; i < da; ++i) X[0][i * da + i] = 1.0;
  for (size_t i = 0; i < db; ++i) Y[0][i * db + i] = 1.0;
  std::vector<double> sig(1, 1.0);  // U = sum_k sig_k X_k (x) Y_k
  auto mul = [](const std::vector<cd>& E, const std::vector<cd>& F, size_t d) { return matmul(E, F, d); };
  auto on_side = [](const Gate& g, const std::vector<int>& S) {
    for (int q : g.q)
      if (std::find(S.begin(), S.end(), q) == S.end()) return false;
    return true;
  };
  // orthonormal Schmidt form of sum_k sig_k X_k (x) Y_k, truncated at tol * s_0
  auto recompress = [&]() {
    const int r = (int)X.size();
    std::vector<cd> Ax(ea * (size_t)r), Ay(eb * (size_t)r);
    for (int k = 0; k < r; ++k) {
      for (size_t e = 0; e < ea; ++e) Ax[e * r + k] = X[k][e] * sig[k];
      for (size_t e = 0; e < eb; ++e) Ay[e * r + k] = Y[k][e];
    }
    // A = U S V^H: column k = sum_i s_i u_i conj(v_i[k])
    Svd sx = jacobi_svd(Ax, (int)ea, r), sy = jacobi_svd(Ay, (int)eb, r);
    auto keep = [](const Svd& s) {
      size_t n = 0;
      while (n < s.s.size() && s.s[n] > 1e-14 * s.s[0]) ++n;
      return n;
    };
    const size_t rx = keep(sx), ry = keep(sy);
    // C_ij = sx_i sy_j sum_k conj(vx_i[k] vy_j[k])
    std::vector<cd> C(rx * ry);
    for (size_t i = 0; i < rx; ++i)
      for (size_t j = 0; j < ry; ++j) {
        cd acc = 0.0;
        for (int k = 0; k < r; ++k) acc += std::conj(sx.v[i][k] * sy.v[j][k]);
        C[i * ry + j] = sx.s[i] * sy.s[j] * acc;
      }
    Svd sc = jacobi_svd(C, (int)rx, (int)ry);  // C = W S Z^H
    std::vector<std::vector<cd>> Xn, Yn;
    std::vector<double> sn;
    const double s0 = sc.s.empty() ? 0.0 : sc.s[0];
    for (size_t m = 0; m < sc.s.size(); ++m) {
      if (!(sc.s[m] > o.svd_rel_tol * s0)) break;
      // U = sum_m s_m (sum_i W_im x^_i) (x) (sum_j conj(Z_jm) y^_j)
      std::vector<cd> xm(ea, 0.0), ym(eb, 0.0);
      for (size_t i = 0; i < rx; ++i)
        for (size_t e = 0; e < ea; ++e) xm[e] += sc.u[m][i] * sx.u[i][e];
      for (size_t j = 0; j < ry; ++j)
        for (size_t e = 0; e < eb; ++e) ym[e] += std::conj(sc.v[m][j]) * sy.u[j][e];
      Xn.push_back(std::move(xm));
      Yn.push_back(std::move(ym));
      sn.push_back(sc.s[m]);
    }
    X.swap(Xn);
    Y.swap(Yn);
    sig.swap(sn);
  };
  for (int gi : u.gids) {
    const Gate& g = gates[gi];
    if (on_side(g, u.Sa)) {
      const std::vector<cd> E = embed(g, u.Sa);
      for (auto& x : X) x = mul(E, x, da);
    } else if (on_side(g, u.Sb)) {
      const std::vector<cd> E = embed(g, u.Sb);
      for (auto& y : Y) y = mul(E, y, db);
    } else {
      // the gate's own Schmidt decomposition across the cut (gate-local
      // index: first-listed qubit = MSB), terms embedded into each side
      std::vector<int> qa, qb, pa, pb;  // its qubits per side and their gate-local bit
      for (int j = 0; j < g.k; ++j) {
        const int bit = g.k - 1 - j;
        if (std::find(u.Sa.begin(), u.Sa.end(), g.q[j]) != u.Sa.end()) {
          qa.push_back(g.q[j]);
          pa.push_back(bit);
        } else {
          qb.push_back(g.q[j]);
          pb.push_back(bit);
        }
      }
      const int ka = (int)qa.size(), kb = (int)qb.size();
      const int ga = 1 << ka, gb = 1 << kb, dg = 1 << g.k;
      auto split = [](int idx, const std::vector<int>& pos) {
        int v = 0;
        for (size_t t = 0; t < pos.size(); ++t) v = (v << 1) | ((idx >> pos[t]) & 1);  // qa[0] = MSB
        return v;
      };
      // M[(ib, jb), (ia, ja)] = G[(i), (j)]
      std::vector<cd> M((size_t)gb * gb * ga * ga, 0.0);
      for (int i = 0; i < dg; ++i)
        for (int j = 0; j < dg; ++j) {
          const int ia = split(i, pa), ib = split(i, pb), ja = split(j, pa), jb = split(j, pb);
          M[(size_t)(ib * gb + jb) * (ga * ga) + (ia * ga + ja)] = g.U[(size_t)i * dg + j];
        }
      Svd sg = jacobi_svd(M, gb * gb, ga * ga);
      std::vector<std::vector<cd>> Xn, Yn;
      std::vector<double> sn;
      for (size_t t = 0; t < sg.s.size(); ++t) {
        if (!(sg.s[t] > 1e-14 * sg.s[0])) break;
        Gate Ga, Gb;  // g^a_t = conj(v_t) as (ia, ja), g^b_t = u_t as (ib, jb), first-listed = MSB
        Ga.k = ka;
        Ga.q = qa;
        Ga.U.resize((size_t)ga * ga);
        for (size_t e = 0; e < Ga.U.size(); ++e) Ga.U[e] = std::conj(sg.v[t][e]);
        Gb.k = kb;
        Gb.q = qb;
        Gb.U.resize((size_t)gb * gb);
        for (size_t e = 0; e < Gb.U.size(); ++e) Gb.U[e] = sg.u[t][e];
        const std::vector<cd> Ea = embed(Ga, u.Sa), Eb = embed(Gb, u.Sb);
        for (size_t k = 0; k < X.size(); ++k) {
          Xn.push_back(mul(Ea, X[k], da));
          Yn.push_back(mul(Eb, Y[k], db));
          sn.push_back(sig[k] * sg.s[t]);
        }
      }
      X.swap(Xn);
      Y.swap(Yn);
      sig.swap(sn);
      recompress();
    }
  }
  recompress();  // (a block without crossing members, or the final form)
  if (sig.empty() || !(sig[0] > 0)) fail(HSF_ERR_INVALID_ARG, "block operator is zero");
  const double sa = std::sqrt((double)da), sb = std::sqrt((double)db);
  for (size_t m = 0; m < sig.size(); ++m) {
    u.sigma.push_back(sig[m]);
    u.c.push_back(cd(sig[m] / (sa * sb), 0.0));
    for (auto& x : X[m]) x *= sa;  // unitary-scale factors (reading 4)
    for (auto& y : Y[m]) y *= sb;
    u.X.push_back(std::move(X[m]));
    u.Y.push_back(std::move(Y[m]));
  }
  u.rank = (int)u.sigma.size();
  u.sequential = true;
}

static void decompose_unit(const std::vector<Gate>& gates, Unit& u, int n_low, const hsf_plan_opts& o) {
  std::set<int> sup;
  for (int gi : u.gids)
    for (int q : gates[gi].q) sup.insert(q);
  u.support.assign(sup.begin(), sup.end());
  for (int q : u.support) (q < n_low ? u.Sb : u.Sa).push_back(q);
  const int nb = (int)u.Sb.size(), na = (int)u.Sa.size(), ks = nb + na;
  u.diag_route = true;
  for (int gi : u.gids) u.diag_route = u.diag_route && gates[gi].diag;
  if (o.analytic_cascades && analytic_cascade(gates, u, n_low, o)) return;
  Svd sv;
  if (u.diag_route) {
    if (ks > 24) fail(HSF_ERR_BLOCK_TOO_LARGE, "diagonal block on more than 24 qubits");
    const size_t N = (size_t)1 << ks;
    std::vector<cd> d(N, 1.0);
    for (int gi : u.gids) {
      const Gate& g = gates[gi];
      std::vector<int> pos(g.k);
      for (int j = 0; j < g.k; ++j)
        pos[j] = (int)(std::find(u.support.begin(), u.support.end(), g.q[j]) - u.support.begin());
      const int dg = 1 << g.k;
      std::vector<cd> diag(dg);
      for (int il = 0; il < dg; ++il) diag[il] = g.U[(size_t)il * dg + il];
      if (g.k == 1) {
        for (size_t i = 0; i < N; ++i) d[i] *= diag[(i >> pos[0]) & 1];
      } else if (g.k == 2) {  // first-listed qubit = MSB of the gate-local index
        for (size_t i = 0; i < N; ++i) d[i] *= diag[(((i >> pos[0]) & 1) << 1) | ((i >> pos[1]) & 1)];
      } else {
        for (size_t i = 0; i < N; ++i) {
          int il = 0;
          for (int j = 0; j < g.k; ++j) il = (il << 1) | (int)((i >> pos[j]) & 1);
          d[i] *= diag[il];
        }
      }
    }
    // M[i^b, i^a] = u(i^a, i^b): the diagonal operator's operator-Schmidt matrix
    const int R = 1 << nb, C = 1 << na;
    std::vector<cd> M((size_t)R * C);
    for (size_t i = 0; i < N; ++i) M[(i & (R - 1)) * C + (i >> nb)] = d[i];
    sv = jacobi_svd(M, R, C);
  } else {
    // sequential route: block_route 2, or auto (0) from 8 support qubits on
    // (dense factors stay <= kMaxDenseQ qubits per side: the device limit)
    const bool seq = o.block_route == 2 || (o.block_route == 0 && ks >= 8);
    if (seq && na <= kMaxDenseQ && nb <= kMaxDenseQ) {
      sequential_unit(gates, u, o);
      return;
    }
    if (ks > o.max_dense_block_qubits)
      fail(HSF_ERR_BLOCK_TOO_LARGE, "dense block on " + std::to_string(ks) + " qubits exceeds max_dense_block_qubits");
    const size_t N = (size_t)1 << ks;
    std::vector<cd> US(N * N, 0.0);
    for (size_t i = 0; i < N; ++i) US[i * N + i] = 1.0;
    for (int gi : u.gids) US = matmul(embed(gates[gi], u.support), US, N);  // later gates on the left
    // Eq. 6: A~[(i^b,j^b),(i^a,j^a)] = U_S[(i^a,i^b),(j^a,j^b)]
    const int R = 1 << (2 * nb), C = 1 << (2 * na);
    const size_t db = (size_t)1 << nb, da = (size_t)1 << na;
    std::vector<cd> At((size_t)R * C);
    for (size_t ia = 0; ia < da; ++ia)
      for (size_t ib = 0; ib < db; ++ib)
        for (size_t ja = 0; ja < da; ++ja)
          for (size_t jb = 0; jb < db; ++jb) {
            size_t row = ((ia << nb) | ib), col = ((ja << nb) | jb);
            At[(ib * db + jb) * C + (ia * da + ja)] = US[row * N + col];
          }
    sv = jacobi_svd(At, R, C);
  }
  // H6: truncation + unitary-scale normalisation
  const double s0 = sv.s.empty() ? 0.0 : sv.s[0];
  if (!(s0 > 0)) fail(HSF_ERR_INVALID_ARG, "block operator is zero");
  const double sa = std::sqrt((double)(1 << na)), sb = std::sqrt((double)(1 << nb));
  for (size_t m = 0; m < sv.s.size(); ++m) {
    if (!(sv.s[m] > o.svd_rel_tol * s0)) break;
    u.sigma.push_back(sv.s[m]);
    u.c.push_back(cd(sv.s[m] / (sa * sb), 0.0));
    // Eq. 8: X_m = sum V*_{m,(i^a,j^a)} |i^a><j^a| ; V*_{m,.} = conj(v_m)
    std::vector<cd> X(sv.v[m].size()), Y(sv.u[m].size());
    for (size_t e = 0; e < X.size(); ++e) X[e] = std::conj(sv.v[m][e]) * sa;
    // Eq. 9: Y_m = sum U_{(i^b,j^b),m} |i^b><j^b|
    for (size_t e = 0; e < Y.size(); ++e) Y[e] = sv.u[m][e] * sb;
    u.X.push_back(std::move(X));
    u.Y.push_back(std::move(Y));
  }
  u.rank = (int)u.sigma.size();
}

// -------------------------------------------------------------- H2 schedule
struct SchedItem {
  bool unit;
  int id;  // gate id or unit id
};

static std::vector<SchedItem> schedule(const std::vector<Gate>& gates, const std::vector<std::vector<int>>& units) {
  const int G = (int)gates.size();
  std::vector<int> owner(G, -1);
  for (size_t u = 0; u < units.size(); ++u)
    for (int gi : units[u]) owner[gi] = (int)u;
  // node ids: units first (0..U-1), then free gates (U + gi)
  const int U = (int)units.size();
  auto node_of = [&](int gi) { return owner[gi] >= 0 ? owner[gi] : U + gi; };
  const int NN = U + G;
  std::vector<std::set<int>> succ(NN);
  std::vector<int> indeg(NN, 0), minid(NN, 1 << 30);
  std::vector<char> exists(NN, 0);
  // dependencies follow commutation: an op depends on every earlier op on a
  // shared qubit unless both are diagonal (diagonal operators commute), so a
  // block of commuting diagonal gates is convex however they are interleaved
  // (the paper reorders commuting RZZ gates to form cascades)
  std::map<int, int> last_nd;             // qubit -> node of the last non-diagonal gate
  std::map<int, std::set<int>> diags;     // qubit -> diagonal nodes since then
  for (int gi = 0; gi < G; ++gi) {
    int nd = node_of(gi);
    exists[nd] = 1;
    minid[nd] = std::min(minid[nd], gi);
    const bool dg = gates[gi].diag;
    std::set<int> deps;
    for (int q : gates[gi].q) {
      auto it = last_nd.find(q);
      if (it != last_nd.end()) deps.insert(it->second);
      if (!dg) {
        auto jt = diags.find(q);
        if (jt != diags.end()) deps.insert(jt->second.begin(), jt->second.end());
      }
    }
    for (int d : deps)
      if (d != nd && succ[d].insert(nd).second) indeg[nd]++;
    for (int q : gates[gi].q) {
      if (dg) {
        diags[q].insert(nd);
      } else {
        last_nd[q] = nd;
        diags[q].clear();
      }
    }
  }
  using P = std::pair<int, int>;
  std::priority_queue<P, std::vector<P>, std::greater<P>> pq;
  int total = 0;
  for (int v = 0; v < NN; ++v)
    if (exists[v]) {
      ++total;
      if (indeg[v] == 0) pq.push({minid[v], v});
    }
  std::vector<SchedItem> order;
  while (!pq.empty()) {
    int v = pq.top().second;
    pq.pop();
    order.push_back(v < U ? SchedItem{true, v} : SchedItem{false, v - U});
    for (int s : succ[v])
      if (--indeg[s] == 0) pq.push({minid[s], s});
  }
  if ((int)order.size() != total)
    fail(HSF_ERR_NONCONVEX_BLOCK, "a block is not convex in the gate-dependency DAG (non-commuting gate inside)");
  return order;
}

// ----------------------------------------------------- H8 half programs
static int64_t push_coef(Plan& P, const std::vector<cd>& v) {
  int64_t off = (int64_t)P.coef.size();
  P.coef.insert(P.coef.end(), v.begin(), v.end());
  return off;
}

// Convert a gate (file order, first-listed = MSB) to an LSB-first op on a half.
static HostOp gate_op(Plan& P, const Gate& g, int first_qubit) {
  HostOp op;
  op.k = g.k;
  op.kind = g.diag ? OP_DIAG : OP_DENSE;
  for (int j = 0; j < g.k; ++j) op.q[j] = g.q[g.k - 1 - j] - first_qubit;  // bit j <- last-listed first
  const int d = 1 << g.k;
  if (g.diag) {
    std::vector<cd> dd(d);
    for (int i = 0; i < d; ++i) dd[i] = g.U[(size_t)i * d + i];
    op.table = push_coef(P, dd);
  } else {
    op.table = push_coef(P, g.U);  // MSB-first local index == LSB-first with reversed q list
  }
  op.stride = 0;
  return op;
}

static std::vector<cd> op_matrix(const Plan& P, const HostOp& op) {
  const size_t d = (size_t)1 << op.k;
  if (op.kind == OP_DIAG) return std::vector<cd>(P.coef.begin() + op.table, P.coef.begin() + op.table + d);
  return std::vector<cd>(P.coef.begin() + op.table, P.coef.begin() + op.table + d * d);
}

// Fusion inside one segment ("gate fusion"): (1) a 1-qubit dense op
// merges into the previous op if that op is a fixed 1-qubit dense op on the
// same qubit and nothing in between touched the qubit; (2) adjacent fixed
// diagonal ops merge while their union has <= kFuseDiagQ qubits (tables of
// <= 256 entries stay L1-resident in the simulator kernels).
constexpr int kFuseDiagQ = 8;

static void fuse_segment(Plan& P, std::vector<HostOp>& seg) {
  // (1)
  std::vector<HostOp> out;
  std::map<int, int> last;  // qubit -> index in out of last op touching it
  for (const HostOp& op : seg) {
    if (op.unit < 0 && op.kind == OP_DENSE && op.k == 1) {
      auto it = last.find(op.q[0]);
      if (it != last.end()) {
        HostOp& prev = out[it->second];
        if (prev.unit < 0 && prev.kind == OP_DENSE && prev.k == 1) {
          auto A = op_matrix(P, op), B = op_matrix(P, prev);
          std::vector<cd> C(4);
          for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) C[i * 2 + j] = A[i * 2 + 0] * B[0 * 2 + j] + A[i * 2 + 1] * B[1 * 2 + j];
          prev.table = push_coef(P, C);
          continue;
        }
      }
    }
    out.push_back(op);
    for (int j = 0; j < op.k; ++j) last[op.q[j]] = (int)out.size() - 1;
  }
  // (2)
  std::vector<HostOp> out2;
  for (const HostOp& op : out) {
    if (!out2.empty() && op.unit < 0 && op.kind == OP_DIAG && out2.back().unit < 0 && out2.back().kind == OP_DIAG) {
      HostOp& prev = out2.back();
      std::set<int> uni(prev.q, prev.q + prev.k);
      uni.insert(op.q, op.q + op.k);
      int runs = 0;
      {
        int prevq = -2;
        for (int q : uni) {
          if (q != prevq + 1) ++runs;
          prevq = q;
        }
      }
      if ((int)uni.size() <= kFuseDiagQ && runs <= 2) {
        std::vector<int> qs(uni.begin(), uni.end());  // ascending
        const int k = (int)qs.size();
        auto Da = op_matrix(P, prev), Db = op_matrix(P, op);
        std::vector<cd> D((size_t)1 << k);
        for (size_t i = 0; i < D.size(); ++i) {
          int ia = 0, ib = 0;
          for (int j = 0; j < prev.k; ++j) {
            int pos = (int)(std::find(qs.begin(), qs.end(), prev.q[j]) - qs.begin());
            ia |= (int)((i >> pos) & 1) << j;
          }
          for (int j = 0; j < op.k; ++j) {
            int pos = (int)(std::find(qs.begin(), qs.end(), op.q[j]) - qs.begin());
            ib |= (int)((i >> pos) & 1) << j;
          }
          D[i] = Da[ia] * Db[ib];
        }
        HostOp f;
        f.kind = OP_DIAG;
        f.k = k;
        for (int j = 0; j < k; ++j) f.q[j] = qs[j];
        f.table = push_coef(P, D);
        prev = f;
        continue;
      }
    }
    out2.push_back(op);
  }
  seg.swap(out2);
}

// Greedy tile-pass planner for halves larger than the SMEM-resident limit.
// Tile = 2^t amplitudes with tile qubits T (always 0..4 for 256 B coalesced
// rows).  A dense op joins the pass if its qubits fit in T (|T| <= t); a
// diagonal op joins regardless of T (its non-tile bits are fixed per tile);
// an op touching a qubit already deferred is deferred (order is preserved).
static DevOp to_dev(const HostOp& op, const std::vector<int>* T) {
  DevOp d{};
  d.kind = op.kind;
  d.k = op.k;
  for (int j = 0; j < op.k; ++j)
    d.q[j] = (T && op.kind == OP_DENSE) ? (int)(std::find(T->begin(), T->end(), op.q[j]) - T->begin()) : op.q[j];
  d.radix = 1;
  d.table = op.table;
  d.stride = op.stride;
  d.div = op.unit;  // unit id until resolved per transition
  return d;
}

struct PassChoice {
  std::vector<int> T;          // ascending tile qubits
  std::vector<int64_t> take;   // op indices (into H.ops) applied in this pass
};

static std::vector<PassChoice> greedy_passes(const Half& H, int64_t ob, int64_t oe, int t) {
  const int low = 5;
  std::vector<PassChoice> out;
  std::vector<int64_t> pending;
  for (int64_t i = ob; i < oe; ++i) pending.push_back(i);
  do {
    std::set<int> T;
    for (int i = 0; i < low; ++i) T.insert(i);
    std::set<int> blocked;
    std::vector<int64_t> take, rest;
    for (int64_t oi : pending) {
      const HostOp& op = H.ops[oi];
      bool blk = false;
      for (int j = 0; j < op.k; ++j) blk = blk || blocked.count(op.q[j]);
      if (blk) {
        for (int j = 0; j < op.k; ++j) blocked.insert(op.q[j]);
        rest.push_back(oi);
        continue;
      }
      if (op.kind == OP_DIAG) {
        take.push_back(oi);
        continue;
      }
      std::set<int> need = T;
      for (int j = 0; j < op.k; ++j) need.insert(op.q[j]);
      if ((int)need.size() <= t) {
        T = need;
        take.push_back(oi);
      } else {
        for (int j = 0; j < op.k; ++j) blocked.insert(op.q[j]);
        rest.push_back(oi);
      }
    }
    if (take.empty() && !pending.empty()) fail(HSF_ERR_UNSUPPORTED, "pass planner made no progress");
    for (int q = 0; q < H.m && (int)T.size() < t; ++q) T.insert(q);
    out.push_back({std::vector<int>(T.begin(), T.end()), take});
    pending.swap(rest);
  } while (!pending.empty());
  return out;
}

// Tile size of a transition's passes: the fewest passes over t in [t, t_max]
// (tile_qubits == 0 => auto: 12, or 13 for complex64 = 64 KiB tiles); each
// pass is an HBM/L2 round trip of every node.
static std::vector<PassChoice> choose_passes(const Half& H, int64_t ob, int64_t oe, int t, int t_max, int& bt) {
  std::vector<PassChoice> best;
  bt = t;
  for (int t2 = t; t2 <= t_max && t2 <= H.m; ++t2) {
    std::vector<PassChoice> c = greedy_passes(H, ob, oe, t2);
    if (best.empty() || c.size() < best.size()) {
      best.swap(c);
      bt = t2;
    }
  }
  return best;
}

static void plan_passes(Half& H, Transition& tr, int64_t ob, int64_t oe, int t, int t_max) {
  int bt = t;
  std::vector<PassChoice> best = choose_passes(H, ob, oe, t, t_max, bt);
  for (auto& pc : best) {
    Pass p;
    p.t = bt;
    p.T = pc.T;  // ascending: tile positions 0..4 are qubits 0..4
    p.op_begin = (int64_t)H.dev_ops.size();
    for (int64_t oi : pc.take) H.dev_ops.push_back(to_dev(H.ops[oi], &p.T));
    p.op_end = (int64_t)H.dev_ops.size();
    tr.passes.push_back(std::move(p));
  }
}

// Register passes: maximal runs of 1-qubit dense ops on at most kRegQ distinct
// tile qubits, interleaved with diagonal ops, become one OP_RPASS whose ops the
// kernel applies to 2^kRegQ amplitudes kept in registers per thread (one SMEM
// round trip for the whole run instead of one sweep + barrier per gate).
static std::vector<DevOp> regpass_rewrite(const std::vector<DevOp>& ops, int t) {
  if (t < kRegQ) return ops;
  std::vector<DevOp> out;
  int hdr = -1;
  std::vector<int> RS;
  size_t free_start = 0;  // out[free_start..) are standalone diagonals (no group owns them)
  auto close = [&]() {
    if (hdr < 0) return;
    int n_r1 = 0;
    for (size_t j = hdr + 1; j < out.size(); ++j) n_r1 += out[j].kind == OP_R1;
    if (n_r1 < 2) {
      // a single 1-qubit gate: a plain SMEM sweep is cheaper than a register
      // pass and keeps the pass on the light kernel variant
      for (size_t j = hdr + 1; j < out.size(); ++j)
        if (out[j].kind == OP_R1) {
          out[j].kind = OP_DENSE;
          out[j].q[0] = RS[out[j].q[0]];
        }
      out.erase(out.begin() + hdr);
      hdr = -1;
      RS.clear();
      free_start = out.size();
      return;
    }
    DevOp& h = out[hdr];
    for (int q = 0; q < t && (int)RS.size() < kRegQ; ++q)
      if (std::find(RS.begin(), RS.end(), q) == RS.end()) RS.push_back(q);
    h = DevOp{};
    h.kind = OP_RPASS;
    h.k = (int)out.size() - hdr - 1;
    for (int j = 0; j < kRegQ; ++j) h.q[j] = RS[j];
    h.radix = 1;
    h.div = 1;
    hdr = -1;
    RS.clear();
    free_start = out.size();
  };
  for (const DevOp& d : ops) {
    if (hdr >= 0 && (int)out.size() - hdr >= kMaxPassOps / 2) close();
    if (d.kind == OP_DENSE && d.k == 1) {
      const int pos = d.q[0];
      auto it = std::find(RS.begin(), RS.end(), pos);
      if (hdr >= 0 && it == RS.end() && (int)RS.size() == kRegQ) close();
      if (hdr < 0) {
        // open the group before the standalone diagonals just preceding it:
        // they run on the registers too (index from the group base + register
        // bits), saving an element-owner SMEM sweep and a barrier
        hdr = (int)std::max(free_start, out.size());
        while ((size_t)hdr > free_start && out[hdr - 1].kind == OP_DIAG) --hdr;
        out.insert(out.begin() + hdr, DevOp{});
      }
      it = std::find(RS.begin(), RS.end(), pos);
      int slot = (int)(it - RS.begin());
      if (it == RS.end()) RS.push_back(pos);
      DevOp r = d;
      r.kind = OP_R1;
      r.q[0] = slot;
      out.push_back(r);
    } else if (d.kind == OP_DIAG) {
      out.push_back(d);
    } else {
      close();
      out.push_back(d);
      free_start = out.size();
    }
  }
  close();
  return out;
}

// ops per kernel pass (<= kMaxPassOps, all staged in SMEM): a long op chain
// on a narrow level becomes several kernels of smaller code, each an L2
// round trip of a few MB -- c3's root passes (127 ops, instruction-fetch
// bound) at 40: 0.578 -> 0.542-0.553 ms (32 / 40 / 48 / 64 / 80 / 128:
// 0.54 / 0.55 / 0.55 / 0.56 / 0.57 / 0.58); c5, q32-1 unchanged. Tiled passes only.
// HSF_MAX_PASS_OPS=n overrides (n >= 128: no split below kMaxPassOps).
static size_t max_pass_ops() {
  static const size_t v = [] {
    const char* e = std::getenv("HSF_MAX_PASS_OPS");
    const long x = e ? std::atol(e) : 40;
    return (size_t)(x > 0 && x < kMaxPassOps ? x : kMaxPassOps);
  }();
  return v;
}

static void finalize_half(Half& H, size_t elem_bytes) {
  std::vector<DevOp> out;
  H.n_passes = 0;
  for (auto& tr : H.trans) {
    std::vector<Pass> np;
    for (const Pass& p : tr.passes) {
      std::vector<DevOp> ops(H.dev_ops.begin() + p.op_begin, H.dev_ops.begin() + p.op_end);
      std::vector<DevOp> rw = regpass_rewrite(ops, p.t);
      // split into kernel passes of <= kMaxPassOps ops without cutting a register pass
      size_t i = 0;
      do {
        Pass q = p;
        q.op_begin = (int64_t)out.size();
        size_t n = 0;
        while (i < rw.size()) {
          size_t w = (rw[i].kind == OP_RPASS) ? (size_t)rw[i].k + 1 : 1;
          // (tiled passes only: splitting a whole-state K1 pass costs a
          // relaunch and an SMEM reload of the state -- c2's half A 0.903 vs
          // 0.907 ms)
          const size_t cap = p.t < H.m ? max_pass_ops() : (size_t)kMaxPassOps;
          if (n + w > cap && n > 0) break;
          for (size_t j = 0; j < w; ++j) out.push_back(rw[i + j]);
          n += w;
          i += w;
        }
        q.op_end = (int64_t)out.size();
        q.heavy = false;
        for (int64_t oi = q.op_begin; oi < q.op_end; ++oi)
          q.heavy = q.heavy || out[oi].kind == OP_RPASS || (out[oi].kind == OP_DENSE && out[oi].k > 2);
        // stage small diagonal tables of this pass in SMEM (bank-spread LDS
        // gathers instead of scattered L1 wavefronts)
        q.tbl_elems = 0;
        for (int64_t oi = q.op_begin; oi < q.op_end; ++oi) {
          DevOp& d = out[oi];
          d.soff = -1;
          // (room for the generated kernels' padded layout x + x/16)
          const int64_t sz = (1 << d.k) + ((1 << d.k) >> 4);
          if (d.kind == OP_DIAG && d.k <= kSmemTableQ && (size_t)(q.tbl_elems + sz) * elem_bytes <= (size_t)kSmemTableBytes) {
            d.soff = (int32_t)q.tbl_elems;
            q.tbl_elems += sz;
          }
        }
        np.push_back(q);
      } while (i < rw.size());
    }
    tr.passes.swap(np);
    H.n_passes += (int)tr.passes.size();
  }
  H.dev_ops.swap(out);
}

// Head fold: while every op of half h so far has kept a qubit in a
// computational-basis state (diagonal gates, or monomial gates -- one nonzero
// per column, e.g. X -- on basis qubits), a diagonal Schmidt factor on basis
// qubits multiplies the half state by the scalar F_{u,d}[bits].  Returns the
// number v0 of leading units whose half-h factors are such scalars, and each
// one's diagonal index (LSB = smallest support qubit).  Exact: the factor acts
// on alpha |b>.
static int head_units(const Plan& P, int h, const std::vector<SchedItem>& order, std::vector<int64_t>& idx) {
  const int first = (h == 0) ? P.n_low : 0, m = (h == 0) ? P.n - P.n_low : P.n_low;
  std::vector<char> cls(m, 1);
  std::vector<int> bit(m, 0);
  std::vector<char> cand(P.units.size(), 0);
  idx.assign(P.units.size(), 0);
  for (const SchedItem& it : order) {
    if (it.unit) {
      const Unit& u = P.units[it.id];
      const std::vector<int>& S = (h == 0) ? u.Sa : u.Sb;
      bool all = true;
      for (int q : S) all = all && cls[q - first];
      if (u.diag_route && all) {
        cand[it.id] = 1;
        int64_t x = 0;
        for (size_t j = 0; j < S.size(); ++j) x |= (int64_t)bit[S[j] - first] << j;
        idx[it.id] = x;
      } else if (!u.diag_route) {
        for (int q : S) cls[q - first] = 0;
      }
      continue;
    }
    const Gate& g = P.gates[it.id];
    bool mine = true;
    for (int q : g.q) mine = mine && ((h == 0) ? q >= P.n_low : q < P.n_low);
    if (!mine || g.diag) continue;
    bool all = true;
    for (int q : g.q) all = all && cls[q - first];
    // monomial: exactly one nonzero per column
    const int D = 1 << g.k;
    int col_row = -1;
    bool mono = all;
    if (all) {
      int b = 0;  // gate-local input index, q[0] = MSB
      for (int j = 0; j < g.k; ++j) b = (b << 1) | bit[g.q[j] - first];
      int nz = 0;
      for (int r = 0; r < D; ++r)
        if (g.U[(size_t)r * D + b] != cd(0)) {
          ++nz;
          col_row = r;
        }
      for (int c = 0; c < D && mono; ++c) {
        int n = 0;
        for (int r = 0; r < D; ++r) n += g.U[(size_t)r * D + c] != cd(0);
        mono = n == 1;
      }
      mono = mono && nz == 1;
    }
    if (mono) {
      for (int j = 0; j < g.k; ++j) bit[g.q[j] - first] = (col_row >> (g.k - 1 - j)) & 1;
    } else {
      for (int q : g.q) cls[q - first] = 0;
    }
  }
  int v0 = 0;
  while (v0 < (int)P.units.size() && cand[v0]) ++v0;
  return v0;
}

// Builds half h's path-tree program over the first U_tree units (U_tree <
// n_units only for the trailing-diagonal fold, whose dropped units carry no
// gate after them).
// Factor ops of a pass evaluated at output level L: the digit of unit u is
// (node / prod_{u < v < L} r_v) % r_u; diagonal qubit lists as <= 3 runs.
static void resolve_digits(Half& H, Pass& p, const std::vector<int32_t>& R, int L) {
  for (int64_t i = p.op_begin; i < p.op_end; ++i) {
    DevOp& d = H.dev_ops[i];
    int unit = (int)d.div;
    if (unit >= 0) {
      d.radix = R[unit];
      d.div = (int64_t)range_prod(R, unit + 1, L);
    } else {
      d.radix = 1;
      d.div = 1;
    }
    // contiguous runs of the diagonal's qubit list (index bit j <- q[j])
    d.nruns = 0;
    if (d.kind == OP_DIAG) {
      int r = 0;
      for (int j = 0; j < d.k;) {
        int e = j + 1;
        while (e < d.k && d.q[e] == d.q[e - 1] + 1) ++e;
        if (r < 3) {
          d.rshift[r] = (uint8_t)d.q[j];
          d.rlen[r] = (uint8_t)(e - j);
          d.roff[r] = (uint8_t)j;
        }
        ++r;
        j = e;
      }
      d.nruns = (r <= 3) ? r : 0;
    }
  }
}

static void build_half(Plan& P, int h, const std::vector<SchedItem>& order, int U_tree, Half& H, int v0 = 0) {
  const int n_low = P.n_low;
  // units [0, v0) are scalars on this half (head fold, see head_units): no
  // factor op, radix 1 in this tree
  std::vector<int32_t> R = P.ranks;
  for (int u = 0; u < v0 && u < (int)R.size(); ++u) R[u] = 1;
  H.first_qubit = (h == 0) ? n_low : 0;
  H.m = (h == 0) ? P.n - n_low : n_low;
  if (H.m > 30) fail(HSF_ERR_UNSUPPORTED, "half-states above 30 qubits are not supported (32-bit device indexing)");
  const int U = U_tree;
  H.last_gate_level = 0;
  // segments.  Factor of unit u opens segment u+1.  With hoisting (default),
  // each local gate goes to the EARLIEST level its dependencies allow: it
  // must follow every earlier op on a shared qubit that it does not commute
  // with (commuting = both diagonal); a factor pins level u+1.  A gate that
  // commutes with a unit's factors (disjoint support, or both diagonal) thus
  // runs once per prefix node above that unit instead of once per child --
  // the same circuit (every reordering swaps commuting operators only),
  // evaluated on fewer path-tree nodes.
  std::vector<std::vector<HostOp>> segs(U + 1);
  std::vector<HostOp> factors(U);
  int level = 0;
  const bool hoist = P.opts.hoist_gates != 0;
  std::vector<int> last_nd(H.m, 0), diag_max(H.m, 0);  // per half-local qubit
  auto dep_level = [&](const HostOp& op) {
    int l = 0;
    for (int j = 0; j < op.k; ++j) {
      l = std::max(l, last_nd[op.q[j]]);
      if (op.kind != OP_DIAG) l = std::max(l, diag_max[op.q[j]]);
    }
    return l;
  };
  auto record = [&](const HostOp& op, int l) {
    for (int j = 0; j < op.k; ++j) {
      if (op.kind == OP_DIAG) {
        diag_max[op.q[j]] = std::max(diag_max[op.q[j]], l);
      } else {
        last_nd[op.q[j]] = l;
        diag_max[op.q[j]] = l;
      }
    }
  };
  for (const SchedItem& it : order) {
    if (it.unit && (it.id >= U_tree || it.id < v0)) continue;  // folded trailing / head-scalar unit
    if (it.unit) {
      const Unit& u = P.units[it.id];
      const std::vector<int>& S = (h == 0) ? u.Sa : u.Sb;
      const auto& F = (h == 0) ? u.X : u.Y;
      HostOp op;
      op.k = (int)S.size();
      op.kind = u.diag_route ? OP_DIAG : OP_DENSE;
      if (op.kind == OP_DENSE && op.k > kMaxDenseQ)
        fail(HSF_ERR_BLOCK_TOO_LARGE, "dense Schmidt factor on more than 5 qubits of one half");
      if (op.kind == OP_DIAG && op.k > kMaxOpQ) fail(HSF_ERR_BLOCK_TOO_LARGE, "diagonal factor on more than 13 qubits");
      for (int j = 0; j < op.k; ++j) op.q[j] = S[j] - H.first_qubit;  // ascending = LSB-first
      op.unit = it.id;
      op.table = (int64_t)P.coef.size();
      for (const auto& f : F) P.coef.insert(P.coef.end(), f.begin(), f.end());
      op.stride = (int64_t)F[0].size();
      factors[it.id] = op;
      level = it.id + 1;
      if (dep_level(op) > level) fail(HSF_ERR_INVALID_ARG, "internal: factor below its dependencies");
      record(op, level);
    } else {
      const Gate& g = P.gates[it.id];
      bool low = true, high = true;
      for (int q : g.q) {
        low = low && q < n_low;
        high = high && q >= n_low;
      }
      if ((h == 0 && high) || (h == 1 && low)) {
        HostOp op = gate_op(P, g, H.first_qubit);
        if (op.kind == OP_DENSE && op.k > kMaxDenseQ) fail(HSF_ERR_UNSUPPORTED, "dense local gate on more than 5 qubits");
        if (op.kind == OP_DIAG && op.k > kMaxOpQ) fail(HSF_ERR_UNSUPPORTED, "diagonal local gate on more than 13 qubits");
        const int l = hoist ? dep_level(op) : level;
        if (l > U) fail(HSF_ERR_INVALID_ARG, "internal: gate below a folded unit");
        record(op, l);
        segs[l].push_back(op);
        H.last_gate_level = std::max(H.last_gate_level, l);
      }
    }
  }
  if (P.opts.fuse_gates)
    for (auto& s : segs) fuse_segment(P, s);
  // flatten: seg_0, F_0, seg_1, ..., F_{U-1}, seg_U
  H.ops.clear();
  H.seg_end.assign(U + 1, 0);
  for (int l = 0; l <= U; ++l) {
    if (l > v0) H.ops.push_back(factors[l - 1]);  // head-scalar units have no factor op
    for (auto& op : segs[l]) H.ops.push_back(op);
    H.seg_end[l] = (int64_t)H.ops.size();
  }
  // Materialised levels (node states written to HBM/L2; the others are
  // recomputed on chip by their children): chosen by dynamic programming over
  // the levels with a per-transition cost model --
  //   launches x 3 us + state bytes / 5 TB/s + wide diagonal table bytes /
  //   15 TB/s (L2) + amplitude-ops / 2.5e13 FMA/s,
  // where a transition a -> b writes every level-b node once per pass, reads
  // its level-a parent (siblings mostly hit L2) and re-applies all ops of the
  // skipped levels per child.  The leaves (level U) are always materialised.
  // K1 tier: the whole half state in one CTA's shared memory (2^14 complex64
  // = 128 KiB of the 227 KiB; 2^13 complex128)
  int smem_limit = (P.opts.dtype == HSF_C64) ? 14 : 13;
  if (const char* e = std::getenv("HSF_SMEM_LIMIT")) smem_limit = std::atoi(e) - (P.opts.dtype == HSF_C64 ? 0 : 1);
  const int t = std::min(H.m, P.opts.tile_qubits > 0 ? P.opts.tile_qubits : 12);
  const int t_max = (P.opts.tile_qubits == 0 && P.opts.dtype == HSF_C64) ? 13 : t;
  // (tile_qubits > 0 below m forces the tiled tier: tests, tile sweeps)
  const bool whole_fits = H.m <= smem_limit && !(P.opts.tile_qubits > 0 && P.opts.tile_qubits < H.m);
  // 2^14 complex64 (128 KiB: one CTA per SM) is K1 only where the cost model
  // prefers it to tiles; smaller halves always are (3+ CTAs per SM)
  const int k1_always = (P.opts.dtype == HSF_C64) ? 13 : 12;
  bool whole = whole_fits;
  auto run_dp = [&](bool whole) {
    const double elem = (P.opts.dtype == HSF_C64) ? 8.0 : 16.0;
    const double amps = std::ldexp(1.0, H.m), S = amps * elem;
    auto nodes = [&](int l) { return (double)range_prod(R, 0, l); };
    auto cost = [&](int a, int b) {
      const int64_t ob = (a < 0) ? 0 : H.seg_end[a], oe = H.seg_end[b];
      size_t np = 1;
      int tt = H.m;
      const double Nb = nodes(b), Na = (a < 0) ? 0.0 : nodes(a);
      if (!whole) np = choose_passes(H, ob, oe, t, t_max, tt).size();
      double bytes = 0;
      for (size_t i = 0; i < np; ++i) {
        const double rd = (i == 0) ? ((a < 0) ? 0.0 : S * (Na + 0.3 * (Nb - Na))) : S * Nb;
        bytes += rd + S * Nb;
      }
      double fma = 0, table = 0;
      const double tiles = std::ldexp(1.0, H.m - tt);
      for (int64_t i = ob; i < oe; ++i) {
        const HostOp& op = H.ops[i];
        if (op.kind == OP_DIAG) {
          fma += 6;
          if (op.k > kSmemTableQ) table += Nb * tiles * std::ldexp(1.0, std::min(op.k, tt)) * elem;
        } else {
          fma += 4.0 * std::ldexp(1.0, op.k);
        }
      }
      // narrow levels run on few SMs: the op chain's throughput scales with
      // CTAs; a 128 KiB whole state is one 8-warp CTA per SM (about half the
      // issue rate of the tiled passes' 3-4 CTAs)
      const bool big = whole && H.m > k1_always;
      const double par = std::min(1.0, Nb * tiles / ((big ? 1.0 : 2.0) * 148)) * (big ? 0.5 : 1.0);
      return 3e-6 * (double)np + bytes / 5e12 + table / 15e12 + fma * amps * Nb / (2.5e13 * par);
    };
    std::vector<double> best(U + 1, 1e300);
    std::vector<int> from(U + 1, -1);
    for (int b2 = 0; b2 <= U; ++b2) {
      best[b2] = cost(-1, b2);
      from[b2] = -1;
      for (int a2 = 0; a2 < b2; ++a2) {
        const double c = best[a2] + cost(a2, b2);
        if (c < best[b2]) {
          best[b2] = c;
          from[b2] = a2;
        }
      }
    }
    std::vector<int> mat;
    for (int l = U; l >= 0; l = from[l]) mat.push_back(l);
    std::reverse(mat.begin(), mat.end());
    return std::make_pair(best[U], mat);
  };
  {
    auto r = run_dp(whole);
    if (whole && H.m > k1_always && P.opts.smem_tier != 1) {
      auto rt = run_dp(false);
      if (std::getenv("HSF_DEBUG_PLAN"))
        std::fprintf(stderr, "K1 tier 2^%d: whole %.3f ms vs tiled %.3f ms\n", H.m, r.first * 1e3, rt.first * 1e3);
      if (rt.first < r.first) {
        whole = false;
        r = rt;
      }
    }
    H.materialized = r.second;
    H.est_ms = r.first * 1e3;
  }
  // transitions + passes
  H.trans.clear();
  H.dev_ops.clear();
  H.n_passes = 0;
  int prev = -1;
  for (int L : H.materialized) {
    Transition tr;
    tr.level_in = prev;
    tr.level_out = L;
    int64_t ob = (prev < 0) ? 0 : H.seg_end[prev];
    int64_t oe = H.seg_end[L];
    if (whole) {
      Pass p;
      p.t = H.m;
      for (int i = 0; i < H.m; ++i) p.T.push_back(i);
      p.op_begin = (int64_t)H.dev_ops.size();
      for (int64_t oi = ob; oi < oe; ++oi) H.dev_ops.push_back(to_dev(H.ops[oi], nullptr));
      p.op_end = (int64_t)H.dev_ops.size();
      tr.passes.push_back(p);
    } else {
      plan_passes(H, tr, ob, oe, t, t_max);
    }
    // resolve factor digits for this transition's output level
    for (auto& p : tr.passes) resolve_digits(H, p, R, L);
    H.trans.push_back(std::move(tr));
    prev = L;
  }
  finalize_half(H, P.opts.dtype == HSF_C64 ? 8 : 16);
  // algorithmic traffic of the tree: every pass reads and writes each output
  // node's state once (the first pass from |0...0> reads nothing)
  H.tree_bytes = 0;
  H.tree_flops = 0;
  {
    const double S = std::ldexp(1.0, H.m) * (P.opts.dtype == HSF_C64 ? 8.0 : 16.0);
    for (const auto& tr : H.trans) {
      const double N = (double)range_prod(R, 0, tr.level_out);
      H.tree_bytes += N * S * (2.0 * (double)tr.passes.size() - (tr.level_in < 0 ? 1.0 : 0.0));
      // FP32/FP64 flops per amplitude (FMA = 2): a dense k-qubit op 8 * 2^k
      // (2^k complex multiply-adds per output amplitude), a 1-qubit gate of a
      // register pass 16, a diagonal 6 (one complex multiply)
      double fl = 0;
      for (const auto& ps : tr.passes)
        for (int64_t i = ps.op_begin; i < ps.op_end; ++i) {
          const DevOp& d = H.dev_ops[i];
          fl += d.kind == OP_DENSE ? 8.0 * std::ldexp(1.0, d.k) : d.kind == OP_R1 ? 16.0 : d.kind == OP_DIAG ? 6.0 : 0.0;
        }
      H.tree_flops += N * std::ldexp(1.0, H.m) * fl;
    }
  }
  // T-leaf variant (see Half::tleaf): the last transition's ops over tiles of
  // 2^10 amplitudes in ONE pass, its R = 2 / 4 / 8 leaves per parent
  // evaluated by one CTA (R x 8 KiB of staging)
  H.tleaf.reset();
  H.tleaf_R = 0;
  if (!whole && H.m >= 10 && !H.trans.empty() && H.trans.back().level_in >= 0) {
    const int lin = H.trans.back().level_in;
    const uint64_t Rc = range_prod(R, lin, U);
    const int64_t ob = H.seg_end[lin], oe = H.seg_end[U];
    if (Rc == 2 || Rc == 4 || Rc == 8) {
      std::vector<PassChoice> pcs = greedy_passes(H, ob, oe, 10);
      if (pcs.size() == 1) {
        auto TL = std::make_shared<Half>();
        TL->m = H.m;
        TL->first_qubit = H.first_qubit;
        Pass p;
        p.t = 10;
        p.T = pcs[0].T;
        p.op_begin = 0;
        for (int64_t oi : pcs[0].take) TL->dev_ops.push_back(to_dev(H.ops[oi], &p.T));
        p.op_end = (int64_t)TL->dev_ops.size();
        resolve_digits(*TL, p, R, U);
        Transition tr;
        tr.level_in = lin;
        tr.level_out = U;
        tr.passes.push_back(p);
        TL->trans.push_back(tr);
        finalize_half(*TL, P.opts.dtype == HSF_C64 ? 8 : 16);
        if (TL->trans[0].passes.size() == 1) {
          H.tleaf = TL;
          H.tleaf_R = (int)Rc;
        }
      }
    }
  }
  if (std::getenv("HSF_DEBUG_PLAN")) {
    static const char* kn[] = {"DENSE", "DIAG", "RPASS", "R1"};
    std::fprintf(stderr, "half %c: m=%d levels=%zu est=%.3f ms\n", h == 0 ? 'A' : 'B', H.m, H.materialized.size(), H.est_ms);
    for (auto& tr : H.trans) {
      std::fprintf(stderr, " trans %d->%d passes=%zu\n", tr.level_in, tr.level_out, tr.passes.size());
      for (auto& p : tr.passes) {
        std::fprintf(stderr, "  pass t=%d tbl=%lld:", p.t, (long long)p.tbl_elems);
        for (int64_t i = p.op_begin; i < p.op_end; ++i) {
          const DevOp& d = H.dev_ops[i];
          std::fprintf(stderr, " %s%s(k%d q", kn[d.kind], d.radix > 1 ? "*" : "", d.k);
          for (int j = 0; j < std::min(d.k, 4); ++j) std::fprintf(stderr, "%s%d", j ? "," : "", d.q[j]);
          std::fprintf(stderr, ")");
        }
        std::fprintf(stderr, "\n");
      }
    }
  }
}

static uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

// ------------------------------------------------------ automatic joint blocks
// The paper groups commuting RZZ gates into cascades sharing one qubit and
// cuts each cascade jointly ("we use a brute force algorithm to reassemble
// cascades of RZZ gates which can be cut jointly"; a cascade of
// diagonal two-qubit gates with a common qubit has Schmidt rank <= 2, Eq. 11,
// P:197-207).  Here: every diagonal two-qubit gate crossing the cut is an
// edge between its low-side and high-side qubit, each endpoint tagged with
// its "epoch" (number of non-diagonal gates on that qubit before the gate,
// so a cascade never spans a non-commuting gate on its shared qubit).  A
// minimum vertex cover of this bipartite multigraph (Koenig: from a maximum
// matching) gives the fewest cascades covering every such gate; each gate
// joins the cascade of a covering endpoint.  Cascades of one gate stay
// separate cuts; other crossing gates are cut individually.
static std::vector<std::vector<int>> auto_blocks(const std::vector<Gate>& gates, int n_low) {
  std::map<std::pair<int, int>, int> lid, rid;  // (qubit, epoch) -> vertex id
  std::vector<std::pair<int, int>> edges;       // (left vertex, right vertex) per candidate gate
  std::vector<int> egate;
  std::map<int, int> epoch;
  for (int gi = 0; gi < (int)gates.size(); ++gi) {
    const Gate& g = gates[gi];
    if (g.k == 2 && g.diag && ((g.q[0] < n_low) != (g.q[1] < n_low))) {
      const int b = std::min(g.q[0], g.q[1]), a = std::max(g.q[0], g.q[1]);
      auto kb = std::make_pair(b, epoch[b]), ka = std::make_pair(a, epoch[a]);
      if (!lid.count(kb)) lid[kb] = (int)lid.size();
      if (!rid.count(ka)) rid[ka] = (int)rid.size();
      edges.push_back({lid[kb], rid[ka]});
      egate.push_back(gi);
    }
    if (!g.diag)
      for (int q : g.q) epoch[q]++;
  }
  const int NL = (int)lid.size(), NR = (int)rid.size();
  std::vector<std::vector<int>> adj(NL);
  for (auto& e : edges) adj[e.first].push_back(e.second);
  for (auto& v : adj) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  // maximum matching (Kuhn's augmenting paths; graphs here have <= ~100 vertices)
  std::vector<int> matchR(NR, -1), matchL(NL, -1);
  std::vector<char> seen;
  std::function<bool(int)> augment = [&](int l) -> bool {
    for (int r : adj[l]) {
      if (seen[r]) continue;
      seen[r] = 1;
      if (matchR[r] < 0 || augment(matchR[r])) {
        matchR[r] = l;
        matchL[l] = r;
        return true;
      }
    }
    return false;
  };
  for (int l = 0; l < NL; ++l) {
    seen.assign(NR, 0);
    augment(l);
  }
  // Koenig: Z = vertices reachable from unmatched left vertices by alternating paths
  std::vector<char> zl(NL, 0), zr(NR, 0);
  std::vector<int> stack;
  for (int l = 0; l < NL; ++l)
    if (matchL[l] < 0) {
      zl[l] = 1;
      stack.push_back(l);
    }
  while (!stack.empty()) {
    int l = stack.back();
    stack.pop_back();
    for (int r : adj[l])
      if (!zr[r] && matchL[l] != r) {
        zr[r] = 1;
        int l2 = matchR[r];
        if (l2 >= 0 && !zl[l2]) {
          zl[l2] = 1;
          stack.push_back(l2);
        }
      }
  }
  // cover = (L \ Z) u (R n Z); each gate joins a covering endpoint (left first)
  std::map<std::pair<int, int>, std::vector<int>> groups;  // (side, vertex) -> gates
  for (size_t i = 0; i < edges.size(); ++i) {
    const int l = edges[i].first, r = edges[i].second;
    if (!zl[l])
      groups[{0, l}].push_back(egate[i]);
    else
      groups[{1, r}].push_back(egate[i]);
  }
  std::vector<std::vector<int>> blocks;
  for (auto& kv : groups)
    if (kv.second.size() >= 2) blocks.push_back(kv.second);
  std::sort(blocks.begin(), blocks.end());
  return blocks;
}

// ----------------------------------------------------------------- driver
Plan* build_plan(const char* text, size_t len, int n_low, int64_t n_blocks, const int64_t* off, const int64_t* ids,
                 const hsf_plan_opts& opts) {
  auto P = std::make_unique<Plan>();
  P->opts = opts;
  const bool dbg = std::getenv("HSF_DEBUG_PLAN_TIME") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "plan %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  P->gates = parse(text, len, &P->n);
  lap("parse");
  P->n_low = n_low;
  if (n_low < 1 || n_low >= P->n) fail(HSF_ERR_INVALID_ARG, "n_low must satisfy 1 <= n_low < n");
  // arbitrary partition: relabel so half B is [0, n_low)
  P->relabel.resize(P->n);
  for (int q = 0; q < P->n; ++q) P->relabel[q] = q;
  if (opts.partition_b) {
    if (P->n < 64 && (opts.partition_b >> P->n))
      fail(HSF_ERR_INVALID_ARG, "partition_b names a qubit beyond the circuit");
    if (__builtin_popcountll(opts.partition_b) != n_low)
      fail(HSF_ERR_INVALID_ARG, "popcount(partition_b) must equal n_low");
    int nb = 0, na = n_low;
    for (int q = 0; q < P->n; ++q) P->relabel[q] = ((opts.partition_b >> q) & 1ull) ? nb++ : na++;
    for (int q = 0; q < P->n; ++q) P->permuted = P->permuted || P->relabel[q] != q;
    for (auto& g : P->gates)
      for (int& q : g.q) q = P->relabel[q];
  }
  const int G = (int)P->gates.size();
  auto crossing = [&](int gi) {
    bool lo = false, hi = false;
    for (int q : P->gates[gi].q) (q < n_low ? lo : hi) = true;
    return lo && hi;
  };
  // units: user blocks (joint mode) + singleton crossing gates
  std::vector<std::vector<int>> units;
  std::vector<char> in_block(G, 0);
  std::vector<std::vector<int>> found;
  if (!opts.individual && n_blocks < 0) {
    found = auto_blocks(P->gates, n_low);
    n_blocks = 0;
  }
  if (!opts.individual && !found.empty()) {
    for (auto& blk : found) {
      for (int gi : blk) in_block[gi] = 1;
      units.push_back(blk);
    }
  }
  if (!opts.individual && n_blocks > 0) {
    if (!off || !ids) fail(HSF_ERR_INVALID_ARG, "block CSR arrays are NULL");
    for (int64_t b = 0; b < n_blocks; ++b) {
      if (off[b + 1] < off[b]) fail(HSF_ERR_INVALID_ARG, "block offsets not monotone");
      std::vector<int> blk;
      for (int64_t e = off[b]; e < off[b + 1]; ++e) {
        int64_t gi = ids[e];
        if (gi < 0 || gi >= G) fail(HSF_ERR_INVALID_ARG, "block gate id out of range");
        if (in_block[gi]) fail(HSF_ERR_INVALID_ARG, "gate in two blocks");
        in_block[gi] = 1;
        blk.push_back((int)gi);
      }
      if (blk.empty()) continue;
      std::sort(blk.begin(), blk.end());
      units.push_back(blk);
    }
  }
  for (int gi = 0; gi < G; ++gi)
    if (!in_block[gi] && crossing(gi)) units.push_back({gi});
  auto order = schedule(P->gates, units);
  lap("schedule");
  // renumber units in schedule order
  std::vector<int> remap(units.size(), -1);
  int nu = 0;
  for (auto& it : order)
    if (it.unit) {
      remap[it.id] = nu;
      P->units.emplace_back();
      P->units.back().gids = units[it.id];
      it.id = nu++;
    }
  // H3-H6
  double log2_np = 0;
  for (auto& u : P->units) {
    decompose_unit(P->gates, u, n_low, opts);
    log2_np += std::log2((double)u.rank);
  }
  // individual-cut count n_p^t: product of the individual crossing-gate ranks
  lap("decompose");
  P->log2_individual = 0;
  {
    hsf_plan_opts o2 = opts;
    for (int gi = 0; gi < G; ++gi)
      if (crossing(gi)) {
        Unit tmp;
        tmp.gids = {gi};
        decompose_unit(P->gates, tmp, n_low, o2);
        P->log2_individual += std::log2((double)tmp.rank);
      }
  }
  lap("individual");
  // H7
  if (log2_np > opts.log2_path_budget + 1e-9)
    fail(HSF_ERR_PATH_BUDGET, "n_p = 2^" + std::to_string(log2_np) + " exceeds the path budget");
  P->n_paths = 1;
  P->sigma_off.push_back(0);
  for (auto& u : P->units) {
    P->n_paths *= (uint64_t)u.rank;
    P->ranks.push_back(u.rank);
    P->unit_analytic.push_back(u.analytic ? 1 : 0);
    P->unit_sequential.push_back(u.sequential ? 1 : 0);
    P->sa.push_back((int32_t)u.Sa.size());
    P->sb.push_back((int32_t)u.Sb.size());
    P->sigmas.insert(P->sigmas.end(), u.sigma.begin(), u.sigma.end());
    P->sigma_off.push_back((int64_t)P->sigmas.size());
  }
  // H8
  const int U = (int)P->units.size();
  build_half(*P, 0, order, U, P->half[0]);
  lap("half A");
  build_half(*P, 1, order, U, P->half[1]);
  lap("half B");
  // Trailing-diagonal fold (bitstring runs): when the last units are all
  // diagonal and no gate follows them in either half (after hoisting), their
  // factors commute to the end of both half-circuits, so for an output sample
  // s = (i_A, i_B) the sum over their Schmidt terms collapses to a scalar:
  //   amp(s) = [prod_u sum_d c_{u,d} X_{u,d}(i_A) Y_{u,d}(i_B)] * sum_{p'} c_p' A_p'(i_A) B_p'(i_B)
  // and the bracket is the block's diagonal D_u evaluated at s's support bits
  // (P:104-109 regrouped).  The path tree then stops at level u0.
  P->fold_u0 = -1;
  if (opts.fold_trailing_diag && U > 0 && P->n <= 63) {
    int u0 = std::max({P->half[0].last_gate_level, P->half[1].last_gate_level, U - kMaxFoldUnits});
    for (int u = U - 1; u >= u0; --u)
      if (!P->units[u].diag_route || P->units[u].support.size() > 16) {
        u0 = u + 1;
        break;
      }
    if (u0 < U) {
      P->fold_u0 = u0;
      P->fold_T = range_prod(P->ranks, u0, U);
      build_half(*P, 0, order, u0, P->half_fold[0]);
      build_half(*P, 1, order, u0, P->half_fold[1]);
      for (int u = u0; u < U; ++u) {
        const Unit& un = P->units[u];
        const int ka = (int)un.Sa.size(), kb = (int)un.Sb.size();
        uint64_t mask = 0;
        for (int q : un.support) mask |= 1ull << q;
        P->trail_mask.push_back(mask);
        P->trail_off.push_back((int64_t)P->trail_tab.size());
        for (size_t x = 0; x < ((size_t)1 << (ka + kb)); ++x) {
          const size_t xb = x & (((size_t)1 << kb) - 1), xa = x >> kb;
          cd v = 0;
          for (int d = 0; d < un.rank; ++d) v += un.c[d] * un.X[d][xa] * un.Y[d][xb];
          P->trail_tab.push_back(v);
        }
      }
    }
  }
  // Half-sided trailing fold (full-output runs on the tensor cores): when the
  // last units' half-h factors are diagonal and no gate of half h follows them
  // (after hoisting), they commute to the end of half h's circuit, so half h's
  // leaf of path p is its leaf of the prefix path p / T times the product of
  // those diagonals at the amplitude's support bits (P:104-109 with the
  // factors moved last).  Half h's tree then stops at level u0 and the
  // product is taken while the split-bf16 GEMM operand is written.
  // The operand prep takes the folded diagonals' product from a per-plan table
  // W[p mod T][i] (one load per element), so the fold reaches as far as that
  // table stays small (kTailTableEntries; c2's half A: 8 of 12 units, T = 256,
  // 8 MiB -- measured 0.880 vs 0.890 ms with the 1-3 unit folds of a 16 MiB
  // prefix-leaf budget), or the shallowest level the half's gates allow.
  //
  // Head fold (same runs): leading units whose half-h factors act on basis
  // qubits are scalars on half h (head_units); they leave half h's tree
  // (radix 1) and their scalars F_{u,d}[bits] join c_p.  Half h's leaf of
  // path p is then its tree leaf ((p / T) mod Tt) -- e.g. c2's half B, whose
  // factors all precede its QFT on the X-prepared basis state, is one state.
  if (opts.fold_trailing_diag && U > 0) {
    const double elem = (opts.dtype == HSF_C64) ? 8.0 : 16.0;
    double budget = kTailPrefixBytes;
    const char* budget_env = std::getenv("HSF_TAIL_PREFIX_BYTES");
    if (budget_env) budget = std::strtod(budget_env, nullptr);  // tests: 0 => longest fold
    const char* nh = std::getenv("HSF_NO_HEAD_FOLD");
    for (int hh = 0; hh < 2; ++hh) {
      std::vector<int64_t> hidx;
      int v0 = (nh && nh[0] == '1') ? 0 : head_units(*P, hh, order, hidx);
      Half tmp;
      const Half* base = &P->half[hh];
      if (v0 > 0) {
        build_half(*P, hh, order, U, tmp, v0);
        base = &tmp;
      }
      std::vector<int32_t> R = P->ranks;
      for (int u = 0; u < v0; ++u) R[u] = 1;
      // default: the longest tail whose weight table W[T][2^m] (one load per
      // operand element, built once per plan) stays within kTailTableEntries;
      // HSF_TAIL_PREFIX_BYTES: the deepest level whose prefix leaves fit that budget
      int u_fit = 0;
      if (budget_env) {
        for (int u = 1; u < U; ++u)
          if ((double)range_prod(R, 0, u) * std::ldexp(elem, P->half[hh].m) <= budget) u_fit = u;
      } else {
        u_fit = U;
        for (int u = U - 1; u >= 0; --u)
          if ((double)range_prod(P->ranks, u, U) * std::ldexp(1.0, P->half[hh].m) <= kTailTableEntries) u_fit = u;
        u_fit = std::min(u_fit, U - 1);
      }
      int u0 = std::max({base->last_gate_level, U - kMaxTail, u_fit, v0});
      for (int u = U - 1; u >= u0; --u)
        if (!P->units[u].diag_route) {
          u0 = u + 1;
          break;
        }
      if (u0 >= U && v0 == 0) continue;
      Plan::Tail& T = P->tail[hh];
      T.u0 = u0;
      T.v0 = v0;
      T.T = range_prod(P->ranks, u0, U);
      T.Tt = range_prod(P->ranks, v0, u0);
      if (u0 == U && v0 > 0)
        T.half = std::move(tmp);
      else
        build_half(*P, hh, order, u0, T.half, v0);
      const int first = P->half[hh].first_qubit;
      for (int u = u0; u < U; ++u) {
        const Unit& un = P->units[u];
        const std::vector<int>& S = hh == 0 ? un.Sa : un.Sb;
        const auto& F = hh == 0 ? un.X : un.Y;
        uint32_t mask = 0;
        for (int q : S) mask |= 1u << (q - first);
        T.mask.push_back(mask);
        T.radix.push_back(un.rank);
        T.off.push_back((int64_t)P->tail_tab.size());
        for (const auto& f : F) P->tail_tab.insert(P->tail_tab.end(), f.begin(), f.end());
      }
      // head scalars: hs[u][d] = F_{u,d}[bits at the factor]
      for (int u = 0; u < v0; ++u) {
        const Unit& un = P->units[u];
        const auto& F = hh == 0 ? un.X : un.Y;
        std::vector<cd> sc(un.rank);
        for (int d = 0; d < un.rank; ++d) sc[d] = F[d][(size_t)hidx[u]];
        T.head.push_back(sc);
      }
    }
  }
  // hash
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, &P->n, sizeof(int));
  h = fnv(h, &P->n_low, sizeof(int));
  for (int s = 0; s < 2; ++s) {
    h = fnv(h, P->half[s].dev_ops.data(), P->half[s].dev_ops.size() * sizeof(DevOp));
    h = fnv(h, P->half_fold[s].dev_ops.data(), P->half_fold[s].dev_ops.size() * sizeof(DevOp));
  }
  h = fnv(h, P->trail_tab.data(), P->trail_tab.size() * sizeof(cd));
  for (int s = 0; s < 2; ++s) h = fnv(h, P->tail[s].half.dev_ops.data(), P->tail[s].half.dev_ops.size() * sizeof(DevOp));
  h = fnv(h, P->tail_tab.data(), P->tail_tab.size() * sizeof(cd));
  for (int s = 0; s < 2; ++s)
    for (const auto& v : P->tail[s].head) h = fnv(h, v.data(), v.size() * sizeof(cd));
  h = fnv(h, P->relabel.data(), P->relabel.size() * sizeof(int));
  h = fnv(h, P->coef.data(), P->coef.size() * sizeof(cd));
  h = fnv(h, P->ranks.data(), P->ranks.size() * sizeof(int32_t));
  P->hash = h;
  return P.release();
}

}  // namespace hsf
