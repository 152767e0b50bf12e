// ldsolver_oracle.cpp -- CPU ORACLE for the LDSolver coarse-grid rollout step, plain C++.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library (through oracle/cpp_oracle.py).  The product path
// (paper_2507_01975_b200) never loads it, and it shares no code, header, table or constant
// generator with the CUDA path.  It restates the step in the order of PAPER.md and of the readings
// listed in DESIGN.md §2 (R1-R23 of SURVEY.md §8c), in plain loops, templated on the number type
// (double = the reference; float = a diagnostic fp32 variant), built -O2 without -ffast-math.
// Batch elements are independent: std::thread workers take whole elements when the batch covers
// the threads, otherwise the rows of every conv layer / FFT pass are split over the threads.
//
// Citations: P:n = /root/reference/PAPER.md line n.  Grid: [0, L)^2, N x N cells, h = L/N, cell
// (i, j) centred at ((i+1/2)h, (j+1/2)h), i = x (fastest), j = y, periodic; fields [B][2][N][N].
//
// Pinned by tests/test_cpp_oracle.py (the same closed forms, invariants and brute-force checks as
// the numpy oracle's pins, plus element-wise agreement with oracle/ldsolver_oracle.py).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

extern "C" {
typedef struct {
  int32_t n, batch;
  double length;
  int32_t system;   // 0 Burgers (gamma = 1/2, no projection; R9), 1 incompressible NS
  double nu, dt;
  int32_t rk_order;   // 2 Heun, 3 SSP-RK3 (Shu-Osher), 4 classical (R13)
  double force_amp, force_k, drag;
  int32_t n_layers, width, activation;   // activation 0 ReLU, 1 exact-erf GELU (R6)
  int32_t tc_head, tc_interval;          // R8
  int32_t stencil_mode;                  // 0 learned net, 1 fixed (w = w_base)
} ora_config;
}

namespace {

thread_local std::string g_err;

// ---------------------------------------------------------------- threads
struct Pool {
  int threads;
  // run f(lo, hi) on `threads` contiguous chunks of [0, n)
  void parallel_for(int n, const std::function<void(int, int)>& f) const {
    const int t = std::max(1, std::min(threads, n));
    if (t == 1) {
      f(0, n);
      return;
    }
    std::vector<std::thread> ws;
    for (int k = 0; k < t; ++k) {
      const int lo = (int)((long long)n * k / t), hi = (int)((long long)n * (k + 1) / t);
      ws.emplace_back([&f, lo, hi]() { f(lo, hi); });
    }
    for (auto& w : ws) w.join();
  }
};

inline int wrap(int i, int n) { return ((i % n) + n) % n; }

// ---------------------------------------------------------------- 1. network (R1, R6)
template <typename R>
struct Net {
  std::vector<int> chans;                 // 2, W, ..., W, n_out
  std::vector<std::vector<R>> W, b;       // W[l][((ky*3 + kx)*ci + c)*co + o] (blob order transposed), b[l][co]
  int act;
};

template <typename R>
R gelu(R x) {   // exact erf form, 1/2 x (1 + erf(x / sqrt 2))
  return (R)0.5 * x * ((R)1 + std::erf(x / std::sqrt((R)2)));
}

// H: [N][N][C] cell-major (index (j*N + i)*C + c); one layer, rows [j0, j1) of the output
template <typename R>
void conv_rows(const std::vector<R>& in, int ci, int N, const std::vector<R>& W, const std::vector<R>& b, int co,
               bool phi, int act, std::vector<R>& out, int j0, int j1) {
  std::vector<R> acc(co);
  for (int j = j0; j < j1; ++j)
    for (int i = 0; i < N; ++i) {
      for (int o = 0; o < co; ++o) acc[o] = b[o];
      for (int ky = 0; ky < 3; ++ky)
        for (int kx = 0; kx < 3; ++kx) {
          // cross-correlation with circular padding: tap (ky, kx) reads cell (i + kx - 1, j + ky - 1)
          const R* x = &in[((size_t)wrap(j + ky - 1, N) * N + wrap(i + kx - 1, N)) * ci];
          for (int c = 0; c < ci; ++c) {
            const R xc = x[c];
            const R* w = &W[((size_t)(ky * 3 + kx) * ci + c) * co];   // W[ky][kx][c][o]
            for (int o = 0; o < co; ++o) acc[o] += w[o] * xc;
          }
        }
      R* y = &out[((size_t)j * N + i) * co];
      for (int o = 0; o < co; ++o) {
        R v = acc[o];
        if (phi) v = act == 1 ? gelu(v) : (v > 0 ? v : (R)0);
        y[o] = v;
      }
    }
}

// R = H_L, H_0 = u (one element, planar [2][N][N]); R: [N][N][n_out]
template <typename R>
void net_forward(const Net<R>& net, const R* u, int N, const Pool& pool, std::vector<R>& Rout) {
  std::vector<R> H((size_t)N * N * 2), G;
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < 2; ++c) H[((size_t)j * N + i) * 2 + c] = u[(size_t)c * N * N + (size_t)j * N + i];
  const int L = (int)net.W.size();
  for (int l = 0; l < L; ++l) {
    const int ci = net.chans[l], co = net.chans[l + 1];
    G.assign((size_t)N * N * co, 0);
    pool.parallel_for(N, [&](int j0, int j1) { conv_rows(H, ci, N, net.W[l], net.b[l], co, l < L - 1, net.act, G, j0, j1); });
    H.swap(G);
  }
  Rout.swap(H);
}

// ---------------------------------------------------------------- 2. constraint (R4, R5)
// w = w_base + Pi R per (axis, op); Pi_I = I - 11^T/6, Pi_D = I - 11^T/6 - s s^T/|s|^2 with the
// tap offsets s = (-2.5, ..., 2.5) (orthogonal projectors: sum w_I fixed, sum w_D and sum s w_D fixed)
template <typename R>
void constrain_cell(const R* raw, const double* base, R* w /*[2][2][6]*/) {
  const double s[6] = {-2.5, -1.5, -0.5, 0.5, 1.5, 2.5};
  double ss = 0;
  for (double v : s) ss += v * v;
  for (int ax = 0; ax < 2; ++ax)
    for (int op = 0; op < 2; ++op) {
      const R* r = raw + (ax * 2 + op) * 6;
      for (int t = 0; t < 6; ++t) {
        R v = 0;
        for (int t2 = 0; t2 < 6; ++t2) {
          double p = (t == t2 ? 1.0 : 0.0) - 1.0 / 6.0;
          if (op == 1) p -= s[t] * s[t2] / ss;
          v += (R)p * r[t2];
        }
        w[(ax * 2 + op) * 6 + t] = (R)base[(ax * 2 + op) * 6 + t] + v;
      }
    }
}

// ---------------------------------------------------------------- 3.-6. tendency (Eq.4; R2, R3, R9, R12)
// w: [N][N][24] (axis, op, tap); T: planar [2][N][N]
template <typename R>
void tendency(const ora_config& c, const R* U, const std::vector<R>& w, R* T) {
  const int N = c.n;
  const R h = (R)(c.length / N), nu = (R)c.nu, gamma = c.system == 0 ? (R)0.5 : (R)1;
  const size_t NN = (size_t)N * N;
  const R* u = U;
  const R* v = U + NN;
  std::vector<R> Fx(2 * NN), Fy(2 * NN);
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) {
      const R* wc = &w[((size_t)j * N + i) * 24];
      // x-face i-1/2 (owned by cell i): taps c(i-3+t, j); y-face j-1/2: taps c(i, j-3+t)
      auto xface = [&](const R* f, const R* st) {
        R s = 0;
        for (int t = 0; t < 6; ++t) s += st[t] * f[(size_t)j * N + wrap(i - 3 + t, N)];
        return s;
      };
      auto yface = [&](const R* f, const R* st) {
        R s = 0;
        for (int t = 0; t < 6; ++t) s += st[t] * f[(size_t)wrap(j - 3 + t, N) * N + i];
        return s;
      };
      const R ux = xface(u, wc + 0);    // face-normal advecting velocities from the interp stencil (R3)
      const R vy = yface(v, wc + 12);
      for (int comp = 0; comp < 2; ++comp) {
        const R* f = comp == 0 ? u : v;
        const R cx = xface(f, wc + 0), dcx = xface(f, wc + 6) / h;
        const R cy = yface(f, wc + 12), dcy = yface(f, wc + 18) / h;
        Fx[comp * NN + (size_t)j * N + i] = gamma * ux * cx - nu * dcx;
        Fy[comp * NN + (size_t)j * N + i] = gamma * vy * cy - nu * dcy;
      }
    }
  const bool src = c.force_amp != 0.0 || c.drag != 0.0;
  for (int comp = 0; comp < 2; ++comp)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) {
        const R* fx = &Fx[comp * NN];
        const R* fy = &Fy[comp * NN];
        R t = -((fx[(size_t)j * N + wrap(i + 1, N)] - fx[(size_t)j * N + i]) +
                (fy[(size_t)wrap(j + 1, N) * N + i] - fy[(size_t)j * N + i])) / h;
        if (src) {
          const R y = ((R)j + (R)0.5) * h;
          if (comp == 0) t += (R)c.force_amp * std::sin((R)c.force_k * y) - (R)c.drag * u[(size_t)j * N + i];
          else t += -(R)c.drag * v[(size_t)j * N + i];
        }
        T[comp * NN + (size_t)j * N + i] = t;
      }
}

// ---------------------------------------------------------------- 7. projection (Eq.13-15; R10, R23)
template <typename R>
void fft1(std::complex<R>* a, int n, int sign) {   // in-place iterative radix-2, X_k = sum_m a_m e^{sign 2 pi i k m / n}
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (int len = 2; len <= n; len <<= 1) {
    for (int k = 0; k < len / 2; ++k) {
      const double ang = sign * 2.0 * M_PI * k / len;
      const std::complex<R> wk((R)std::cos(ang), (R)std::sin(ang));
      for (int s = 0; s < n; s += len) {
        const std::complex<R> x = a[s + k], y = a[s + k + len / 2] * wk;
        a[s + k] = x + y;
        a[s + k + len / 2] = x - y;
      }
    }
  }
}

template <typename R>
void fft2(std::vector<std::complex<R>>& A, int N, int sign, const Pool& pool) {
  pool.parallel_for(N, [&](int j0, int j1) {
    for (int j = j0; j < j1; ++j) fft1(&A[(size_t)j * N], N, sign);
  });
  pool.parallel_for(N, [&](int i0, int i1) {
    std::vector<std::complex<R>> col(N);
    for (int i = i0; i < i1; ++i) {
      for (int j = 0; j < N; ++j) col[j] = A[(size_t)j * N + i];
      fft1(col.data(), N, sign);
      for (int j = 0; j < N; ++j) A[(size_t)j * N + i] = col[j];
    }
  });
}

// U <- U - G_c p, p = -(D_c G_c)^+ D_c U: d = [u(i+1)-u(i-1) + v(j+1)-v(j-1)] / 2h;
// p_hat = -d_hat / (kx^2 + ky^2), k_hat_m = sin(k_m h)/h (k_m = m, or m - N for m >= N/2), with k_hat = 0
// at m = 0 and m = N/2 by index and p_hat = 0 on the four modes mx, my in {0, N/2}.
template <typename R>
void project(const ora_config& c, R* U, const Pool& pool) {
  const int N = c.n;
  const size_t NN = (size_t)N * N;
  const R h = (R)(c.length / N);
  R* u = U;
  R* v = U + NN;
  std::vector<std::complex<R>> A(NN);
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i)
      A[(size_t)j * N + i] = ((u[(size_t)j * N + wrap(i + 1, N)] - u[(size_t)j * N + wrap(i - 1, N)]) +
                              (v[(size_t)wrap(j + 1, N) * N + i] - v[(size_t)wrap(j - 1, N) * N + i])) /
                             ((R)2 * h);
  fft2(A, N, -1, pool);
  std::vector<R> kh(N);
  for (int m = 0; m < N; ++m) {
    const int k = m < N / 2 ? m : m - N;
    kh[m] = (m == 0 || m == N / 2) ? (R)0 : (R)(std::sin(2.0 * M_PI * k / N) / (double)h);
  }
  for (int my = 0; my < N; ++my)
    for (int mx = 0; mx < N; ++mx) {
      const bool null = (mx == 0 || mx == N / 2) && (my == 0 || my == N / 2);
      std::complex<R>& z = A[(size_t)my * N + mx];
      z = null ? std::complex<R>(0) : -z / (kh[mx] * kh[mx] + kh[my] * kh[my]);
    }
  fft2(A, N, +1, pool);
  std::vector<R> p(NN);
  for (size_t q = 0; q < NN; ++q) p[q] = A[q].real() / (R)((double)N * N);
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) {
      u[(size_t)j * N + i] -= (p[(size_t)j * N + wrap(i + 1, N)] - p[(size_t)j * N + wrap(i - 1, N)]) / ((R)2 * h);
      v[(size_t)j * N + i] -= (p[(size_t)wrap(j + 1, N) * N + i] - p[(size_t)wrap(j - 1, N) * N + i]) / ((R)2 * h);
    }
}

// ---------------------------------------------------------------- 8. RK step with per-stage projection (R7, R8, R13)
template <typename R>
struct Solver {
  ora_config c;
  Net<R> net;
  double base[24];
  size_t NN;

  // T(U) on one element; e (if non-null and tc_head) receives R[24:26] of this evaluation
  void T(const R* U, R* Tout, R* e, const Pool& pool) const {
    const int N = c.n;
    std::vector<R> w(NN * 24);
    if (c.stencil_mode == 1) {
      for (size_t q = 0; q < NN; ++q)
        for (int k = 0; k < 24; ++k) w[q * 24 + k] = (R)base[k];
    } else {
      std::vector<R> Rn;
      net_forward(net, U, N, pool, Rn);
      const int no = net.chans.back();
      for (size_t q = 0; q < NN; ++q) constrain_cell(&Rn[q * no], base, &w[q * 24]);
      if (e && c.tc_head)
        for (size_t q = 0; q < NN; ++q) {
          e[q] = Rn[q * no + 24];
          e[NN + q] = Rn[q * no + 25];
        }
    }
    tendency(c, U, w, Tout);
  }
  void P(R* U, const Pool& pool) const {
    if (c.system == 1) project(c, U, pool);
  }

  // one step of one element, in place
  void step(R* u, int64_t k, const Pool& pool) const {
    const size_t F = 2 * NN;
    const R dt = (R)c.dt;
    std::vector<R> T1(F), e(F, 0), Us(F), U2(F), Tk(F);
    T(u, T1.data(), e.data(), pool);   // e from the stage-1 net on u^n (R8)
    const bool add_e = c.tc_head && ((k + 1) % c.tc_interval == 0);
    auto E = [&](size_t q) { return add_e ? e[q] : (R)0; };
    if (c.rk_order == 2) {
      for (size_t q = 0; q < F; ++q) Us[q] = u[q] + dt * T1[q];
      P(Us.data(), pool);
      T(Us.data(), Tk.data(), nullptr, pool);
      for (size_t q = 0; q < F; ++q) u[q] = (R)0.5 * u[q] + (R)0.5 * (Us[q] + dt * Tk[q]) + E(q);
      P(u, pool);
    } else if (c.rk_order == 3) {
      for (size_t q = 0; q < F; ++q) Us[q] = u[q] + dt * T1[q];
      P(Us.data(), pool);
      T(Us.data(), Tk.data(), nullptr, pool);
      for (size_t q = 0; q < F; ++q) U2[q] = (R)0.75 * u[q] + (R)0.25 * (Us[q] + dt * Tk[q]);
      P(U2.data(), pool);
      T(U2.data(), Tk.data(), nullptr, pool);
      for (size_t q = 0; q < F; ++q) u[q] = u[q] / (R)3 + ((R)2 / (R)3) * (U2[q] + dt * Tk[q]) + E(q);
      P(u, pool);
    } else {
      std::vector<R> K(T1);   // K1 + 2 K2 + 2 K3 + K4
      for (size_t q = 0; q < F; ++q) Us[q] = u[q] + (R)0.5 * dt * T1[q];
      P(Us.data(), pool);
      T(Us.data(), Tk.data(), nullptr, pool);
      for (size_t q = 0; q < F; ++q) { K[q] += (R)2 * Tk[q]; Us[q] = u[q] + (R)0.5 * dt * Tk[q]; }
      P(Us.data(), pool);
      T(Us.data(), Tk.data(), nullptr, pool);
      for (size_t q = 0; q < F; ++q) { K[q] += (R)2 * Tk[q]; Us[q] = u[q] + dt * Tk[q]; }
      P(Us.data(), pool);
      T(Us.data(), Tk.data(), nullptr, pool);
      for (size_t q = 0; q < F; ++q) u[q] = u[q] + dt / (R)6 * (K[q] + Tk[q]) + E(q);
      P(u, pool);
    }
  }
};

int validate(const ora_config* c) {
  if (!c) return (g_err = "cfg is NULL", -1);
  if (c->n < 4 || (c->n & (c->n - 1))) return (g_err = "n must be a power of two >= 4", -1);
  if (c->batch < 1 || c->rk_order < 2 || c->rk_order > 4 || c->tc_interval < 1)
    return (g_err = "bad batch / rk_order / tc_interval", -1);
  if (c->stencil_mode == 0 && (c->n_layers < 2 || c->width < 1)) return (g_err = "bad net shape", -1);
  if (c->tc_head && c->stencil_mode != 0) return (g_err = "tc_head needs the learned net", -1);
  return 0;
}

size_t param_count(const ora_config* c) {
  if (c->stencil_mode != 0) return 0;
  const int no = 24 + (c->tc_head ? 2 : 0);
  size_t n = 0;
  for (int l = 0; l < c->n_layers; ++l) {
    const int ci = l == 0 ? 2 : c->width, co = l == c->n_layers - 1 ? no : c->width;
    n += (size_t)co * 9 * ci + co;
  }
  return n;
}

template <typename R>
int make_solver(const ora_config* c, const float* params, size_t n_params, const double* base24, Solver<R>& S) {
  if (validate(c)) return -1;
  S.c = *c;
  S.NN = (size_t)c->n * c->n;
  if (base24) {
    for (int k = 0; k < 24; ++k) S.base[k] = base24[k];
  } else {   // 2nd-order central (R5): interp (0,0,1/2,1/2,0,0), deriv (0,0,-1,1,0,0)
    for (int k = 0; k < 24; ++k) S.base[k] = 0.0;
    for (int ax = 0; ax < 2; ++ax) {
      S.base[ax * 12 + 2] = S.base[ax * 12 + 3] = 0.5;
      S.base[ax * 12 + 6 + 2] = -1.0;
      S.base[ax * 12 + 6 + 3] = 1.0;
    }
  }
  if (c->stencil_mode == 0) {
    if (!params || n_params != param_count(c)) return (g_err = "params NULL or n_params mismatch", -1);
    const int no = 24 + (c->tc_head ? 2 : 0);
    S.net.act = c->activation;
    S.net.chans.push_back(2);
    for (int l = 0; l + 1 < c->n_layers; ++l) S.net.chans.push_back(c->width);
    S.net.chans.push_back(no);
    size_t off = 0;
    for (int l = 0; l < c->n_layers; ++l) {
      const int ci = S.net.chans[l], co = S.net.chans[l + 1];
      std::vector<R> Wl((size_t)co * 9 * ci);   // blob W[co][ky][kx][ci] -> [ky][kx][ci][co]
      for (int o = 0; o < co; ++o)
        for (int tap = 0; tap < 9; ++tap)
          for (int cc = 0; cc < ci; ++cc) Wl[((size_t)tap * ci + cc) * co + o] = (R)params[off + ((size_t)o * 9 + tap) * ci + cc];
      S.net.W.push_back(Wl);
      off += (size_t)co * 9 * ci;
      S.net.b.push_back(std::vector<R>(params + off, params + off + co));
      off += co;
    }
  }
  return 0;
}

int hw_threads(int threads) {
  if (threads > 0) return threads;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

// run f(element, inner_pool) over the batch: whole elements per thread when B >= threads, else
// elements one after another with the threads inside (rows of each conv layer / FFT pass)
void over_batch(int B, int threads, const std::function<void(int, const Pool&)>& f) {
  if (B >= threads && threads > 1) {
    Pool outer{threads}, inner{1};
    outer.parallel_for(B, [&](int b0, int b1) {
      for (int b = b0; b < b1; ++b) f(b, inner);
    });
  } else {
    Pool inner{threads};
    for (int b = 0; b < B; ++b) f(b, inner);
  }
}

template <typename R>
int rollout_t(const ora_config* c, const float* params, size_t n_params, const double* base24, double* u,
              int64_t step_index, int32_t n_steps, int32_t threads, int64_t* bad_step) {
  Solver<R> S;
  if (make_solver(c, params, n_params, base24, S)) return -1;
  const size_t F = 2 * S.NN;
  const int th = hw_threads(threads);
  std::vector<int64_t> bad(c->batch, -1);
  over_batch(c->batch, th, [&](int b, const Pool& pool) {
    std::vector<R> x(u + b * F, u + (b + 1) * F);
    for (int s = 0; s < n_steps && bad[b] < 0; ++s) {
      S.step(x.data(), step_index + s, pool);
      for (size_t q = 0; q < F; ++q)
        if (!std::isfinite((double)x[q])) { bad[b] = step_index + s; break; }
    }
    for (size_t q = 0; q < F; ++q) u[b * F + q] = (double)x[q];
  });
  for (int64_t v : bad)
    if (v >= 0) {
      *bad_step = v;
      g_err = "non-finite field at step " + std::to_string(v);
      return -5;
    }
  return 0;
}

}  // namespace

extern "C" {

const char* ora_last_error(void) { return g_err.c_str(); }
size_t ora_param_count(const ora_config* c) { return validate(c) ? 0 : param_count(c); }
int ora_hardware_threads(void) { return hw_threads(0); }

// n_steps steps of every element of u ([B][2][N][N] fp64, in place), the first one with step index
// step_index (TC gating, R8).  precision 0: fp64 arithmetic; 1: fp32 (inputs / outputs still fp64).
// threads 0: one per hardware thread.  Returns 0, -1 (bad argument, see ora_last_error) or -5
// (non-finite field; *bad_step = its step index).
int ora_rollout(const ora_config* c, const float* params, size_t n_params, const double* base24, double* u,
                int64_t step_index, int32_t n_steps, int32_t threads, int32_t precision, int64_t* bad_step) {
  if (!u || !bad_step || n_steps < 0) return (g_err = "bad arguments", -1);
  *bad_step = -1;
  return precision == 1 ? rollout_t<float>(c, params, n_params, base24, u, step_index, n_steps, threads, bad_step)
                        : rollout_t<double>(c, params, n_params, base24, u, step_index, n_steps, threads, bad_step);
}

// Components (fp64), for the pins: R [B][N][N][n_out] raw net output; w [B][N][N][24] constrained
// stencils; T [B][2][N][N] tendency; P(u) in place (NS projection).
int ora_net(const ora_config* c, const float* params, size_t n_params, const double* u, double* Rout,
            int32_t threads) {
  Solver<double> S;
  if (make_solver(c, params, n_params, nullptr, S)) return -1;
  if (c->stencil_mode != 0) return (g_err = "no net in fixed mode", -1);
  const int no = S.net.chans.back();
  over_batch(c->batch, hw_threads(threads), [&](int b, const Pool& pool) {
    std::vector<double> R;
    net_forward(S.net, u + b * 2 * S.NN, c->n, pool, R);
    std::copy(R.begin(), R.end(), Rout + b * S.NN * no);
  });
  return 0;
}

int ora_stencils(const ora_config* c, const float* params, size_t n_params, const double* base24, const double* u,
                 double* w, int32_t threads) {
  Solver<double> S;
  if (make_solver(c, params, n_params, base24, S)) return -1;
  over_batch(c->batch, hw_threads(threads), [&](int b, const Pool& pool) {
    if (c->stencil_mode == 1) {
      for (size_t q = 0; q < S.NN; ++q)
        for (int k = 0; k < 24; ++k) w[(b * S.NN + q) * 24 + k] = S.base[k];
      return;
    }
    std::vector<double> R;
    net_forward(S.net, u + b * 2 * S.NN, c->n, pool, R);
    const int no = S.net.chans.back();
    for (size_t q = 0; q < S.NN; ++q) constrain_cell(&R[q * no], S.base, &w[(b * S.NN + q) * 24]);
  });
  return 0;
}

int ora_tendency(const ora_config* c, const float* params, size_t n_params, const double* base24, const double* u,
                 double* T, int32_t threads) {
  Solver<double> S;
  if (make_solver(c, params, n_params, base24, S)) return -1;
  over_batch(c->batch, hw_threads(threads), [&](int b, const Pool& pool) {
    S.T(u + b * 2 * S.NN, T + b * 2 * S.NN, nullptr, pool);
  });
  return 0;
}

int ora_project(const ora_config* c, double* u, int32_t threads) {
  if (validate(c)) return -1;
  const size_t NN = (size_t)c->n * c->n;
  over_batch(c->batch, hw_threads(threads), [&](int b, const Pool& pool) { project(*c, u + b * 2 * NN, pool); });
  return 0;
}

}  // extern "C"
