// femgen.cu — row-wise on-device FEM assembly (include/fem_gen.h).
//
// One thread per free DOF ("row").  The thread visits every element incident to
// its node in increasing element order (cell lexicographic, then the split's
// element order), evaluates that element's stiffness row and load entries, and
// accumulates them in a fixed stencil of slots keyed by the neighbour's lattice
// offset; slots are then emitted in ascending free-DOF order.  No scatter, no
// atomics, no sort: the pattern is value-independent (Q7) and the
// row length is known from the enumeration alone.
#include <cub/cub.cuh>

#include <cmath>

#include "common.cuh"
#include "fem_gen.h"

namespace pcgb {
namespace {

struct Geo {
  int fam, c, np, m;  // np: lattice points per axis (incl. boundary), m: free per axis
  int dim, jitter;
  uint64_t seed;
  double h, hs;       // cell size, lattice spacing
};

__host__ __device__ inline Geo make_geo(const fem_spec &s) {
  Geo g;
  g.fam = s.family;
  g.c = s.c;
  g.np = (s.family == FEM_P2_TRI) ? 2 * s.c + 1 : s.c + 1;
  g.m = g.np - 2;
  g.dim = (s.family == FEM_P1_TET) ? 3 : 2;
  g.jitter = s.jitter;
  g.seed = s.seed;
  g.h = 1.0 / s.c;
  g.hs = (s.family == FEM_P2_TRI) ? g.h / 2 : g.h;
  return g;
}

// SplitMix64 output idx of stream seed; uniform in [0,1) from the top 53 bits
__device__ __forceinline__ double u01(uint64_t seed, uint64_t idx) {
  uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ bool on_boundary2(const Geo &g, int a, int b) {
  return a == 0 || b == 0 || a == g.np - 1 || b == g.np - 1;
}

// jittered (pre-repair) coordinates of lattice node (a,b); no FMA contraction so
// that the repair decisions below are taken on exactly rounded values
__device__ __forceinline__ void jittered(const Geo &g, int a, int b, double &x, double &y) {
  x = __dmul_rn((double)a, g.hs);
  y = __dmul_rn((double)b, g.hs);
  if (!g.jitter || on_boundary2(g, a, b)) return;
  const uint64_t id = (uint64_t)a + (uint64_t)g.np * (uint64_t)b;
  const double amp = __dmul_rn(0.3, g.h);
  const double dx = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u01(g.seed, 2 * id)), 1.0), amp);
  const double dy = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u01(g.seed, 2 * id + 1)), 1.0), amp);
  x = __dadd_rn(x, dx);
  y = __dadd_rn(y, dy);
}

// 3D (reading R3): interior nodes move by (2u-1)(0.15h)
// per coordinate, u = SplitMix64(seed, 3*node+axis); for this amplitude every Kuhn
// tet keeps its orientation (volume >= 0.1 of the lattice tet's), so no repair.
__device__ __forceinline__ void node_xyz(const Geo &g, int i, int j, int l, double (&X)[3]) {
  X[0] = (double)i * g.h;
  X[1] = (double)j * g.h;
  X[2] = (double)l * g.h;
  if (!g.jitter || i == 0 || j == 0 || l == 0 || i == g.c || j == g.c || l == g.c) return;
  const uint64_t id = (uint64_t)i + (uint64_t)g.np * ((uint64_t)j + (uint64_t)g.np * (uint64_t)l);
  const double amp = __dmul_rn(0.15, g.h);
#pragma unroll
  for (int ax = 0; ax < 3; ax++)
    X[ax] = __dadd_rn(X[ax], __dmul_rn(__dsub_rn(__dmul_rn(2.0, u01(g.seed, 3 * id + ax)), 1.0), amp));
}

__device__ __forceinline__ double area2_rn(double x0, double y0, double x1, double y1, double x2, double y2) {
  return __dsub_rn(__dmul_rn(__dsub_rn(x1, x0), __dsub_rn(y2, y0)), __dmul_rn(__dsub_rn(x2, x0), __dsub_rn(y1, y0)));
}

// vertices (lattice) of triangle t of cell (ci,cj) in the "/" split (P1 spacing)
__device__ __forceinline__ void tri_verts(int ci, int cj, int t, int (&va)[3], int (&vb)[3]) {
  va[0] = ci; vb[0] = cj;
  if (t == 0) { va[1] = ci + 1; vb[1] = cj; va[2] = ci + 1; vb[2] = cj + 1; }
  else        { va[1] = ci + 1; vb[1] = cj + 1; va[2] = ci; vb[2] = cj + 1; }
}

// final coordinates after the one-pass repair: an interior node is reset to the
// lattice iff some triangle containing it has jittered signed area <= 0
__device__ void node_xy(const Geo &g, int a, int b, double &x, double &y) {
  jittered(g, a, b, x, y);
  if (!g.jitter || on_boundary2(g, a, b)) return;
  for (int cj = b - 1; cj <= b; cj++)
    for (int ci = a - 1; ci <= a; ci++)
      for (int t = 0; t < 2; t++) {
        int va[3], vb[3];
        tri_verts(ci, cj, t, va, vb);
        bool has = false;
        for (int k = 0; k < 3; k++) has |= (va[k] == a && vb[k] == b);
        if (!has) continue;
        double px[3], py[3];
        for (int k = 0; k < 3; k++) jittered(g, va[k], vb[k], px[k], py[k]);
        if (area2_rn(px[0], py[0], px[1], py[1], px[2], py[2]) <= 0.0) {
          x = __dmul_rn((double)a, g.hs);
          y = __dmul_rn((double)b, g.hs);
          return;
        }
      }
}

__device__ __forceinline__ double f_eval(const fem_spec &s, const double *p, const double *ctr, int col) {
  switch (s.fkind) {
    case FEM_F_ONE: return 1.0;
    case FEM_F_SIN2D: return 2.0 * M_PI * M_PI * sinpi(p[0]) * sinpi(p[1]);
    case FEM_F_SIN3D: return 3.0 * M_PI * M_PI * sinpi(p[0]) * sinpi(p[1]) * sinpi(p[2]);
    case FEM_F_BUMP3D: {
      const double dx = p[0] - ctr[3 * col], dy = p[1] - ctr[3 * col + 1], dz = p[2] - ctr[3 * col + 2];
      return exp(-(dx * dx + dy * dy + dz * dz) / (2.0 * s.sigma * s.sigma));
    }
    default: return 0.0;
  }
}

constexpr int MAXK = 32;
constexpr int MAXSLOT = 27;

// ------------------------------------------------------------ per-row assembly
// Accumulates row `r` into slot arrays.  Returns the node's lattice coords.
// val[s] : stiffness sums per neighbour slot; touched[s]: slot in element graph
// bsum[k]: load integrals; for the Dirichlet lift the caller needs neighbour coords.
struct RowAcc {
  double val[MAXSLOT];
  bool touched[MAXSLOT];
  double b[MAXK];
};

__device__ __forceinline__ int slot2(int da, int db, int R) { return (db + R) * (2 * R + 1) + (da + R); }

// 2D P1 (lattice or jittered): elements = triangles of the 4 cells around (a,b)
__device__ void row_p1tri(const fem_spec &s, const Geo &g, int a, int b, bool values, RowAcc &acc) {
  const int c = g.c;
  for (int cj = b - 1; cj <= b; cj++)
    for (int ci = a - 1; ci <= a; ci++) {
      if (ci < 0 || cj < 0 || ci >= c || cj >= c) continue;
      for (int t = 0; t < 2; t++) {
        int va[3], vb[3];
        tri_verts(ci, cj, t, va, vb);
        int me = -1;
        for (int k = 0; k < 3; k++)
          if (va[k] == a && vb[k] == b) me = k;
        if (me < 0) continue;
        for (int k = 0; k < 3; k++) acc.touched[slot2(va[k] - a, vb[k] - b, 1)] = true;
        if (!values) continue;
        double x[3], y[3];
        for (int k = 0; k < 3; k++) node_xy(g, va[k], vb[k], x[k], y[k]);
        const double d = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
        double gx[3], gy[3];
        gx[0] = (y[1] - y[2]) / d; gy[0] = (x[2] - x[1]) / d;
        gx[1] = (y[2] - y[0]) / d; gy[1] = (x[0] - x[2]) / d;
        gx[2] = (y[0] - y[1]) / d; gy[2] = (x[1] - x[0]) / d;
        const double area = fabs(d) * 0.5;
        for (int k = 0; k < 3; k++)
          acc.val[slot2(va[k] - a, vb[k] - b, 1)] += area * (gx[me] * gx[k] + gy[me] * gy[k]);
        // load: midpoints of edges (0,1),(1,2),(0,2); φ_me = λ_me there
        if (s.fkind != FEM_F_ZERO) {
          const int E[3][2] = {{0, 1}, {1, 2}, {0, 2}};
          for (int q = 0; q < 3; q++) {
            const int i0 = E[q][0], i1 = E[q][1];
            if (i0 != me && i1 != me) continue;
            const double p[3] = {0.5 * (x[i0] + x[i1]), 0.5 * (y[i0] + y[i1]), 0.0};
            acc.b[0] += (area / 3.0) * f_eval(s, p, nullptr, 0) * 0.5;
          }
        }
      }
    }
}

// 2D P2: 6-DOF triangles on the half-lattice; (a,b) half-lattice coords
__device__ void row_p2tri(const fem_spec &s, const Geo &g, int a, int b, bool values, RowAcc &acc) {
  const int c = g.c;
  const int ci_lo = (a % 2 == 0) ? a / 2 - 1 : (a - 1) / 2, ci_hi = (a % 2 == 0) ? a / 2 : (a - 1) / 2;
  const int cj_lo = (b % 2 == 0) ? b / 2 - 1 : (b - 1) / 2, cj_hi = (b % 2 == 0) ? b / 2 : (b - 1) / 2;
  for (int cj = cj_lo; cj <= cj_hi; cj++)
    for (int ci = ci_lo; ci <= ci_hi; ci++) {
      if (ci < 0 || cj < 0 || ci >= c || cj >= c) continue;
      const int a0 = 2 * ci, b0 = 2 * cj, a1 = a0 + 2, b1 = b0 + 2;
      for (int t = 0; t < 2; t++) {
        int da[6], db[6];
        if (t == 0) {
          const int A[6] = {a0, a1, a1, a0 + 1, a1, a0 + 1}, B[6] = {b0, b0, b1, b0, b0 + 1, b0 + 1};
          for (int k = 0; k < 6; k++) { da[k] = A[k]; db[k] = B[k]; }
        } else {
          const int A[6] = {a0, a1, a0, a0 + 1, a0 + 1, a0}, B[6] = {b0, b1, b1, b0 + 1, b1, b0 + 1};
          for (int k = 0; k < 6; k++) { da[k] = A[k]; db[k] = B[k]; }
        }
        int me = -1;
        for (int k = 0; k < 6; k++)
          if (da[k] == a && db[k] == b) me = k;
        if (me < 0) continue;
        for (int k = 0; k < 6; k++) acc.touched[slot2(da[k] - a, db[k] - b, 2)] = true;
        if (!values) continue;
        double x[3], y[3];
        for (int k = 0; k < 3; k++) { x[k] = da[k] * g.hs; y[k] = db[k] * g.hs; }
        const double d = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
        double gx[3], gy[3];
        gx[0] = (y[1] - y[2]) / d; gy[0] = (x[2] - x[1]) / d;
        gx[1] = (y[2] - y[0]) / d; gy[1] = (x[0] - x[2]) / d;
        gx[2] = (y[0] - y[1]) / d; gy[2] = (x[1] - x[0]) / d;
        const double area = fabs(d) * 0.5;
        const int E[3][2] = {{0, 1}, {1, 2}, {0, 2}};
        for (int q = 0; q < 3; q++) {  // quadrature point: midpoint of edge q
          double L[3] = {0, 0, 0};
          L[E[q][0]] = 0.5;
          L[E[q][1]] = 0.5;
          double phx[6], phy[6], ph[6];
          for (int v = 0; v < 3; v++) {
            ph[v] = L[v] * (2.0 * L[v] - 1.0);
            phx[v] = (4.0 * L[v] - 1.0) * gx[v];
            phy[v] = (4.0 * L[v] - 1.0) * gy[v];
          }
          for (int e = 0; e < 3; e++) {
            const int i0 = E[e][0], i1 = E[e][1];
            ph[3 + e] = 4.0 * L[i0] * L[i1];
            phx[3 + e] = 4.0 * (L[i0] * gx[i1] + L[i1] * gx[i0]);
            phy[3 + e] = 4.0 * (L[i0] * gy[i1] + L[i1] * gy[i0]);
          }
          const double w = area / 3.0;
          for (int k = 0; k < 6; k++)
            acc.val[slot2(da[k] - a, db[k] - b, 2)] += w * (phx[me] * phx[k] + phy[me] * phy[k]);
          if (s.fkind != FEM_F_ZERO && ph[me] != 0.0) {
            const double p[3] = {0.5 * (x[E[q][0]] + x[E[q][1]]), 0.5 * (y[E[q][0]] + y[E[q][1]]), 0.0};
            acc.b[0] += w * f_eval(s, p, nullptr, 0) * ph[me];
          }
        }
      }
    }
}

// 3D P1 Kuhn: 6 tets in each of the 8 cells around (i,j,l)
__device__ void row_p1tet(const fem_spec &s, const Geo &g, int i, int j, int l, bool values, RowAcc &acc,
                          const double *ctr) {
  const int c = g.c;
  const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const double QA = 0.5854101966249685, QB = 0.1381966011250105;
  for (int cl = l - 1; cl <= l; cl++)
    for (int cj = j - 1; cj <= j; cj++)
      for (int ci = i - 1; ci <= i; ci++) {
        if (ci < 0 || cj < 0 || cl < 0 || ci >= c || cj >= c || cl >= c) continue;
        for (int p = 0; p < 6; p++) {
          int v[4][3];
          v[0][0] = ci; v[0][1] = cj; v[0][2] = cl;
          for (int k = 0; k < 3; k++) {
            v[k + 1][0] = v[k][0]; v[k + 1][1] = v[k][1]; v[k + 1][2] = v[k][2];
            v[k + 1][PERM[p][k]] += 1;
          }
          int me = -1;
          for (int k = 0; k < 4; k++)
            if (v[k][0] == i && v[k][1] == j && v[k][2] == l) me = k;
          if (me < 0) continue;
          for (int k = 0; k < 4; k++) acc.touched[(v[k][2] - l + 1) * 9 + (v[k][1] - j + 1) * 3 + (v[k][0] - i + 1)] = true;
          if (!values) continue;
          double X[4][3];
          for (int k = 0; k < 4; k++) node_xyz(g, v[k][0], v[k][1], v[k][2], X[k]);
          double e[3][3];
          for (int k = 0; k < 3; k++)
            for (int d = 0; d < 3; d++) e[k][d] = X[k + 1][d] - X[0][d];
          // rows of J^{-1}: (e2 x e3, e3 x e1, e1 x e2) / det
          double G[4][3];
          const int CA[3] = {1, 2, 0}, CB[3] = {2, 0, 1};
          for (int k = 0; k < 3; k++) {
            const double *u = e[CA[k]], *w = e[CB[k]];
            G[k + 1][0] = u[1] * w[2] - u[2] * w[1];
            G[k + 1][1] = u[2] * w[0] - u[0] * w[2];
            G[k + 1][2] = u[0] * w[1] - u[1] * w[0];
          }
          const double det = e[0][0] * G[1][0] + e[0][1] * G[1][1] + e[0][2] * G[1][2];
          for (int k = 1; k < 4; k++)
            for (int d = 0; d < 3; d++) G[k][d] /= det;
          for (int d = 0; d < 3; d++) G[0][d] = -(G[1][d] + G[2][d] + G[3][d]);
          const double vol = fabs(det) / 6.0;
          for (int k = 0; k < 4; k++)
            acc.val[(v[k][2] - l + 1) * 9 + (v[k][1] - j + 1) * 3 + (v[k][0] - i + 1)] +=
                vol * (G[me][0] * G[k][0] + G[me][1] * G[k][1] + G[me][2] * G[k][2]);
          if (s.fkind != FEM_F_ZERO) {
            const int kk = s.fkind == FEM_F_BUMP3D ? s.k : 1;
            for (int q = 0; q < 4; q++) {
              double pq[3];
              for (int d = 0; d < 3; d++) {
                double sm = 0.0;
                for (int r = 0; r < 4; r++)
                  if (r != q) sm += X[r][d];
                pq[d] = QA * X[q][d] + QB * sm;
              }
              const double lam = (me == q) ? QA : QB;
              for (int col = 0; col < kk; col++) acc.b[col] += (vol / 4.0) * f_eval(s, pq, ctr, col) * lam;
            }
          }
        }
      }
}

__device__ __forceinline__ double g_eval(const fem_spec &s, double x, double y, double z = 0.0) {
  if (s.gkind == FEM_G_X2MY2) return x * x - y * y;
  if (s.gkind == FEM_G_LINEAR3D) return __dadd_rn(__dsub_rn(__dadd_rn(1.0, __dmul_rn(2.0, x)), __dmul_rn(3.0, y)),
                                                  __dmul_rn(0.5, z));
  return 0.0;
}

// Assemble row r (global free index) into acc, then visit slots in ascending
// column order calling emit(col, val) for kept entries; returns the count.
template <class Emit>
__device__ int build_row(const fem_spec &s, const Geo &g, int64_t r, bool values, const double *ctr, RowAcc &acc,
                         int *bad, Emit emit) {
  for (int t = 0; t < MAXSLOT; t++) {
    acc.val[t] = 0.0;
    acc.touched[t] = false;
  }
  for (int t = 0; t < MAXK; t++) acc.b[t] = 0.0;
  const int m = g.m;
  int cnt = 0;
  if (g.dim == 2) {
    const int a = (int)(r % m) + 1, b = (int)(r / m) + 1;
    const int R = g.fam == FEM_P2_TRI ? 2 : 1;
    if (g.fam == FEM_P2_TRI) row_p2tri(s, g, a, b, values, acc);
    else row_p1tri(s, g, a, b, values, acc);
    const int W = 2 * R + 1;
    for (int db = -R; db <= R; db++)
      for (int da = -R; da <= R; da++) {
        const int t = (db + R) * W + (da + R);
        if (!acc.touched[t]) continue;
        const int na = a + da, nb = b + db;
        if (on_boundary2(g, na, nb)) {  // Dirichlet lift b_F -= K_FB g_B
          if (values && s.gkind != FEM_G_ZERO) {
            double x, y;
            node_xy(g, na, nb, x, y);
            acc.b[0] -= acc.val[t] * g_eval(s, x, y);
          }
          continue;
        }
        if (s.policy == FEM_PAT_AXIS && abs(da) + abs(db) > 1) {
          if (values && acc.val[t] != 0.0) atomicOr(bad, 1);
          continue;
        }
        emit((int64_t)(na - 1) + (int64_t)m * (nb - 1), acc.val[t]);
        cnt++;
      }
  } else {
    const int64_t mm = m;
    const int i = (int)(r % mm) + 1, j = (int)((r / mm) % mm) + 1, l = (int)(r / (mm * mm)) + 1;
    row_p1tet(s, g, i, j, l, values, acc, ctr);
    for (int dl = -1; dl <= 1; dl++)
      for (int dj = -1; dj <= 1; dj++)
        for (int di = -1; di <= 1; di++) {
          const int t = (dl + 1) * 9 + (dj + 1) * 3 + (di + 1);
          if (!acc.touched[t]) continue;
          const int ni = i + di, nj = j + dj, nl = l + dl;
          if (ni == 0 || nj == 0 || nl == 0 || ni == g.c || nj == g.c || nl == g.c) {  // Dirichlet lift
            if (values && s.gkind != FEM_G_ZERO) {
              double Xb[3];
              node_xyz(g, ni, nj, nl, Xb);
              acc.b[0] -= acc.val[t] * g_eval(s, Xb[0], Xb[1], Xb[2]);
            }
            continue;
          }
          if (s.policy == FEM_PAT_AXIS && abs(di) + abs(dj) + abs(dl) > 1) {
            if (values && acc.val[t] != 0.0) atomicOr(bad, 1);
            continue;
          }
          emit((int64_t)(ni - 1) + mm * ((nj - 1) + mm * (int64_t)(nl - 1)), acc.val[t]);
          cnt++;
        }
  }
  return cnt;
}

__global__ void __launch_bounds__(128) count_kernel(fem_spec s, int64_t r0, int64_t r1, int64_t *cnt) {
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  const Geo g = make_geo(s);
  RowAcc acc;
  int dummy = 0;
  cnt[r - r0] = build_row(s, g, r, false, nullptr, acc, &dummy, [](int64_t, double) {});
}

__global__ void __launch_bounds__(128) fill_kernel(fem_spec s, int64_t r0, int64_t r1, const int64_t *__restrict__ rp,
                                                   int64_t *__restrict__ col, double *__restrict__ val,
                                                   double *__restrict__ B, int64_t ldb, const double *ctr, int *bad) {
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  const Geo g = make_geo(s);
  RowAcc acc;
  int64_t k = rp[r - r0];
  build_row(s, g, r, true, ctr, acc, bad, [&](int64_t j, double v) {
    col[k] = j;
    val[k] = v;
    k++;
  });
  if (B) {
    const int kk = s.fkind == FEM_F_BUMP3D ? s.k : 1;
    for (int cidx = 0; cidx < kk; cidx++) B[(r - r0) + (int64_t)cidx * ldb] = acc.b[cidx];
  }
}

__global__ void centres_kernel(uint64_t seed, int k, double *ctr) {
  const int t = threadIdx.x;
  if (t < 3 * k) ctr[t] = u01(seed, (uint64_t)t);  // c_s,axis = U(seed, 3s + axis)
}

// ------------------------------------------------------------ element-by-element triplets
// One thread per element e (cells lexicographic, then the split's element order —
// the row-wise generator's enumeration): its npe x npe stiffness matrix K_e over ALL
// lattice nodes (Neumann, before Dirichlet elimination), emitted as triplets
// (node_a, node_b, K_e[a][b]) at position e * npe^2 + a * npe + b.  coo_to_csr of
// the triplets of every element sums each entry over the elements in element order:
// the assembled stiffness (generic path).
//   P1: K_e = |T| G G^T with G the barycentric gradients (P:78 cot formula, §8(c).3)
//   P2: K_e[a][b] = sum over the 3 edge midpoints q of |T|/3 grad phi_a . grad phi_b
__global__ void __launch_bounds__(128) elem_coo_kernel(fem_spec s, int64_t e0, int64_t e1, int64_t *__restrict__ ro,
                                                       int64_t *__restrict__ co, double *__restrict__ vo) {
  const int64_t e = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e1) return;
  const Geo g = make_geo(s);
  const int64_t np = g.np;
  const size_t o = (size_t)(e - e0);
  if (s.family == FEM_P1_TRI || s.family == FEM_P2_TRI) {
    const int64_t cell = e >> 1;
    const int t = (int)(e & 1);
    const int ci = (int)(cell % g.c), cj = (int)(cell / g.c);
    if (s.family == FEM_P1_TRI) {
      int va[3], vb[3];
      tri_verts(ci, cj, t, va, vb);
      double x[3], y[3];
      for (int k = 0; k < 3; k++) node_xy(g, va[k], vb[k], x[k], y[k]);
      const double d = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
      double gx[3], gy[3];
      gx[0] = (y[1] - y[2]) / d; gy[0] = (x[2] - x[1]) / d;
      gx[1] = (y[2] - y[0]) / d; gy[1] = (x[0] - x[2]) / d;
      gx[2] = (y[0] - y[1]) / d; gy[2] = (x[1] - x[0]) / d;
      const double area = fabs(d) * 0.5;
      for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
          const size_t q = o * 9 + a * 3 + b;
          ro[q] = va[a] + np * vb[a];
          co[q] = va[b] + np * vb[b];
          vo[q] = area * (gx[a] * gx[b] + gy[a] * gy[b]);
        }
    } else {
      const int a0 = 2 * ci, b0 = 2 * cj, a1 = a0 + 2, b1 = b0 + 2;
      int da[6], db[6];
      if (t == 0) {
        const int A[6] = {a0, a1, a1, a0 + 1, a1, a0 + 1}, B[6] = {b0, b0, b1, b0, b0 + 1, b0 + 1};
        for (int k = 0; k < 6; k++) { da[k] = A[k]; db[k] = B[k]; }
      } else {
        const int A[6] = {a0, a1, a0, a0 + 1, a0 + 1, a0}, B[6] = {b0, b1, b1, b0 + 1, b1, b0 + 1};
        for (int k = 0; k < 6; k++) { da[k] = A[k]; db[k] = B[k]; }
      }
      double x[3], y[3];
      for (int k = 0; k < 3; k++) { x[k] = da[k] * g.hs; y[k] = db[k] * g.hs; }
      const double d = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
      double gx[3], gy[3];
      gx[0] = (y[1] - y[2]) / d; gy[0] = (x[2] - x[1]) / d;
      gx[1] = (y[2] - y[0]) / d; gy[1] = (x[0] - x[2]) / d;
      gx[2] = (y[0] - y[1]) / d; gy[2] = (x[1] - x[0]) / d;
      const double w = (fabs(d) * 0.5) / 3.0;
      const int E[3][2] = {{0, 1}, {1, 2}, {0, 2}};
      double K[6][6];
      for (int a = 0; a < 6; a++)
        for (int b = 0; b < 6; b++) K[a][b] = 0.0;
      for (int q = 0; q < 3; q++) {
        double L[3] = {0, 0, 0};
        L[E[q][0]] = 0.5;
        L[E[q][1]] = 0.5;
        double phx[6], phy[6];
        for (int v = 0; v < 3; v++) {
          phx[v] = (4.0 * L[v] - 1.0) * gx[v];
          phy[v] = (4.0 * L[v] - 1.0) * gy[v];
        }
        for (int m = 0; m < 3; m++) {
          const int i0 = E[m][0], i1 = E[m][1];
          phx[3 + m] = 4.0 * (L[i0] * gx[i1] + L[i1] * gx[i0]);
          phy[3 + m] = 4.0 * (L[i0] * gy[i1] + L[i1] * gy[i0]);
        }
        for (int a = 0; a < 6; a++)
          for (int b = 0; b < 6; b++) K[a][b] += w * (phx[a] * phx[b] + phy[a] * phy[b]);
      }
      for (int a = 0; a < 6; a++)
        for (int b = 0; b < 6; b++) {
          const size_t q = o * 36 + a * 6 + b;
          ro[q] = da[a] + np * db[a];
          co[q] = da[b] + np * db[b];
          vo[q] = K[a][b];
        }
    }
    return;
  }
  // P1_TET: Kuhn tet p of cell (ci, cj, cl)
  const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const int64_t cell = e / 6;
  const int p = (int)(e % 6);
  const int ci = (int)(cell % g.c), cj = (int)((cell / g.c) % g.c), cl = (int)(cell / ((int64_t)g.c * g.c));
  int v[4][3];
  v[0][0] = ci; v[0][1] = cj; v[0][2] = cl;
  for (int k = 0; k < 3; k++) {
    v[k + 1][0] = v[k][0]; v[k + 1][1] = v[k][1]; v[k + 1][2] = v[k][2];
    v[k + 1][PERM[p][k]] += 1;
  }
  double X[4][3];
  for (int k = 0; k < 4; k++) node_xyz(g, v[k][0], v[k][1], v[k][2], X[k]);
  double ed[3][3];
  for (int k = 0; k < 3; k++)
    for (int d = 0; d < 3; d++) ed[k][d] = X[k + 1][d] - X[0][d];
  double G[4][3];
  const int CA[3] = {1, 2, 0}, CB[3] = {2, 0, 1};
  for (int k = 0; k < 3; k++) {
    const double *u = ed[CA[k]], *w = ed[CB[k]];
    G[k + 1][0] = u[1] * w[2] - u[2] * w[1];
    G[k + 1][1] = u[2] * w[0] - u[0] * w[2];
    G[k + 1][2] = u[0] * w[1] - u[1] * w[0];
  }
  const double det = ed[0][0] * G[1][0] + ed[0][1] * G[1][1] + ed[0][2] * G[1][2];
  for (int k = 1; k < 4; k++)
    for (int d = 0; d < 3; d++) G[k][d] /= det;
  for (int d = 0; d < 3; d++) G[0][d] = -(G[1][d] + G[2][d] + G[3][d]);
  const double vol = fabs(det) / 6.0;
  for (int a = 0; a < 4; a++)
    for (int b = 0; b < 4; b++) {
      const size_t q = o * 16 + a * 4 + b;
      ro[q] = v[a][0] + np * (v[a][1] + np * (int64_t)v[a][2]);
      co[q] = v[b][0] + np * (v[b][1] + np * (int64_t)v[b][2]);
      vo[q] = vol * (G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2]);
    }
}

pcg_status check_spec(const fem_spec *s) {
  if (!s) return fail(PCG_ERR_INVALID_ARG, "fem: null spec");
  if (s->family < FEM_P1_TRI || s->family > FEM_P2_TRI) return fail(PCG_ERR_INVALID_ARG, "fem: bad family");
  if (s->c < 2) return fail(PCG_ERR_INVALID_ARG, "fem: c must be >= 2");
  if (s->jitter && s->family == FEM_P2_TRI) return fail(PCG_ERR_INVALID_ARG, "fem: jitter needs P1 elements");
  if (s->family == FEM_P1_TET && s->gkind != FEM_G_ZERO && s->gkind != FEM_G_LINEAR3D)
    return fail(PCG_ERR_INVALID_ARG, "fem: 3D supports g = 0 or LINEAR3D");
  if (s->family != FEM_P1_TET && s->gkind == FEM_G_LINEAR3D) return fail(PCG_ERR_INVALID_ARG, "fem: LINEAR3D is 3D");
  if (s->family == FEM_P1_TET && s->jitter && s->policy == FEM_PAT_AXIS)
    return fail(PCG_ERR_INVALID_ARG, "fem: jittered tets need the ELEMENT pattern");
  if (s->fkind == FEM_F_BUMP3D && (s->k < 1 || s->k > MAXK || s->family != FEM_P1_TET))
    return fail(PCG_ERR_INVALID_ARG, "fem: BUMP3D needs P1_TET and 1 <= k <= 32");
  if (s->policy == FEM_PAT_AXIS && (s->family == FEM_P2_TRI))
    return fail(PCG_ERR_INVALID_ARG, "fem: AXIS policy is for lattice P1");
  return PCG_OK;
}

}  // namespace
}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status fem_problem_size(const fem_spec *s, int64_t *n_free, int64_t *nnz_total, int64_t *n_nodes) {
  PCG_TRY(check_spec(s));
  const Geo g = make_geo(*s);
  const int64_t m = g.m, np = g.np;
  int64_t n = 0, nnz = 0;
  if (g.dim == 2) {
    n = m * m;
    if (s->family == FEM_P2_TRI) nnz = 46LL * s->c * s->c - 96LL * s->c + 53;
    else nnz = s->policy == FEM_PAT_AXIS ? 5 * m * m - 4 * m : 7 * m * m - 8 * m + 2;
  } else {
    n = m * m * m;
    nnz = s->policy == FEM_PAT_AXIS ? 7 * m * m * m - 6 * m * m : -1;  // element graph: count on device
  }
  if (n_free) *n_free = n;
  if (nnz_total) *nnz_total = nnz;
  if (n_nodes) *n_nodes = g.dim == 2 ? np * np : np * np * np;
  return PCG_OK;
}

extern "C" pcg_status fem_count(const fem_spec *s, int64_t r0, int64_t r1, int64_t *d_rp, int64_t *nnz_out,
                                void *stream) {
  PCG_TRY(check_spec(s));
  int64_t n;
  fem_problem_size(s, &n, nullptr, nullptr);
  if (r0 < 0 || r1 < r0 || r1 > n || !d_rp || !nnz_out) return fail(PCG_ERR_INVALID_ARG, "fem_count: bad range");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = r1 - r0;
  PCG_CUDA(cudaMemsetAsync(d_rp, 0, sizeof(int64_t) * (rows + 1), st));
  if (rows > 0) {
    count_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(*s, r0, r1, d_rp + 1);
    count_launch();
    PCG_CUDA(cudaGetLastError());
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, d_rp + 1, d_rp + 1, rows, st);
    void *tbuf;
    PCG_CUDA(cudaMallocAsync(&tbuf, tb, st));
    cub::DeviceScan::InclusiveSum(tbuf, tb, d_rp + 1, d_rp + 1, rows, st);
    PCG_CUDA(cudaFreeAsync(tbuf, st));
  }
  PCG_CUDA(cudaMemcpyAsync(nnz_out, d_rp + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}

extern "C" pcg_status fem_assemble(const fem_spec *s, int64_t r0, int64_t r1, int64_t *d_rp, int64_t *d_col,
                                   double *d_val, double *d_B, int64_t ldb, void *stream) {
  PCG_TRY(check_spec(s));
  int64_t n;
  fem_problem_size(s, &n, nullptr, nullptr);
  if (r0 < 0 || r1 < r0 || r1 > n || !d_rp || !d_col || !d_val) return fail(PCG_ERR_INVALID_ARG, "fem_assemble: bad argument");
  if (d_B && ldb < r1 - r0) return fail(PCG_ERR_INVALID_ARG, "fem_assemble: ldb < rows");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = r1 - r0;
  double *ctr;
  int *bad;
  PCG_CUDA(cudaMallocAsync(&ctr, sizeof(double) * 3 * MAXK, st));
  PCG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  PCG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  centres_kernel<<<1, 3 * MAXK, 0, st>>>(s->seed, s->fkind == FEM_F_BUMP3D ? s->k : 0, ctr);
  count_launch();
  if (rows > 0) {
    fill_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(*s, r0, r1, d_rp, d_col, d_val, d_B, ldb, ctr, bad);
    count_launch();
    PCG_CUDA(cudaGetLastError());
  }
  int h_bad = 0;
  PCG_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaFreeAsync(ctr, st));
  PCG_CUDA(cudaFreeAsync(bad, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  if (h_bad) return fail(PCG_ERR_INVALID_ARG, "fem_assemble: AXIS policy dropped a nonzero entry");
  return PCG_OK;
}

extern "C" pcg_status fem_element_count(const fem_spec *s, int64_t *n_elem, int32_t *npe, int64_t *n_nodes) {
  PCG_TRY(check_spec(s));
  const Geo g = make_geo(*s);
  const int64_t c = s->c;
  if (n_elem) *n_elem = s->family == FEM_P1_TET ? 6 * c * c * c : 2 * c * c;
  if (npe) *npe = s->family == FEM_P1_TET ? 4 : (s->family == FEM_P2_TRI ? 6 : 3);
  if (n_nodes) *n_nodes = s->family == FEM_P1_TET ? (int64_t)g.np * g.np * g.np : (int64_t)g.np * g.np;
  return PCG_OK;
}

extern "C" pcg_status fem_element_coo(const fem_spec *s, int64_t e0, int64_t e1, int64_t *d_row, int64_t *d_col,
                                      double *d_val, void *stream) {
  PCG_TRY(check_spec(s));
  int64_t ne = 0;
  fem_element_count(s, &ne, nullptr, nullptr);
  if (e0 < 0 || e1 < e0 || e1 > ne || ((!d_row || !d_col || !d_val) && e1 > e0))
    return fail(PCG_ERR_INVALID_ARG, "fem_element_coo: bad element range or null output");
  cudaStream_t st = (cudaStream_t)stream;
  if (e1 > e0) {
    elem_coo_kernel<<<(unsigned)((e1 - e0 + 127) / 128), 128, 0, st>>>(*s, e0, e1, d_row, d_col, d_val);
    count_launch();
    PCG_CUDA(cudaGetLastError());
  }
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}
