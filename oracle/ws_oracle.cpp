// =====================================================================================
//  ws_oracle.cpp — the ORACLE of arXiv 2410.08946 "Parallel Watershed Partitioning".
//
//  TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded, fp64.  Only tests/,
//  __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
//  it.  It shares NO code, header, table or constant with the CUDA path
//  (paper_2410_08946_b200/csrc) and never includes anything from it.
//
//  Citation keys: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
//  Cn = reading n of SURVEY.md §8(c) (restated in DESIGN.md "Readings").
//
//  What it computes (each a plain DEFINITION, written out; no blocking/fusion):
//    oracle_gradient   O1+O2  blur (C8) + gradient magnitude (C9) + quantise (C10)
//    oracle_watershed  O3+O4  steepest-descent pointers (Eq. 1), BFS plateau
//                             distances + max-index parent (C5/C6),
//                             regions = voxels reaching the same regional minimum,
//                             canonical label = min voxel index (C7)
//    oracle_waterfall  O6+O7  RAG with per-pair min pass height (Alg. 4 l.2-7),
//                             strict edge order K (C14), Boruvka levels (C13)
//    oracle_waterfall_u16  O12  O6+O7 on a 16-bit image (NEXT f4)
//    oracle_waterfall_reconstruct  O9  the paper-literal waterfall: newmin + image raise
//                             (Alg. 4 steps V-VI), watershed re-run per layer (Alg. 5)
//  Pins (tests/test_oracle_*.py): SciPy/NumPy for O1-O2, closed forms, the paper's worked
//  examples, literal Alg. 1 on exhaustive tiny images, Kruskal-MST
//  waterfall, invariants.  No function here is "parity unpinned".
// =====================================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <utility>
#include <vector>

namespace {

// Grid: ndim==2 -> n0 independent images of n1 x n2 (no adjacency along axis 0, C18);
//       ndim==3 -> one volume n0 x n1 x n2.  Row-major, last axis fastest (C1).
struct Grid {
  int ndim;
  int64_t n0, n1, n2;
  int64_t N() const { return n0 * n1 * n2; }
  int64_t idx(int64_t z, int64_t y, int64_t x) const { return (z * n1 + y) * n2 + x; }
};

// N(p): in-bounds neighbours a unit step away, p excluded, clipped at the border
// (C2).  Returned in increasing linear-index order.
struct Nb {
  int64_t v[26];
  int n = 0;
  const int64_t* begin() const { return v; }
  const int64_t* end() const { return v + n; }
  bool empty() const { return n == 0; }
};

Nb neighbours(const Grid& g, int conn, int64_t p) {
  Nb out;
  int64_t x = p % g.n2, y = (p / g.n2) % g.n1, z = p / (g.n1 * g.n2);
  int zr = (g.ndim == 3) ? 1 : 0;  // 2D images: no neighbour across axis 0
  for (int dz = -zr; dz <= zr; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (dz == 0 && dy == 0 && dx == 0) continue;
        int l1 = std::abs(dz) + std::abs(dy) + std::abs(dx);
        if ((conn == 4 || conn == 6) && l1 != 1) continue;  // von Neumann
        int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if (zz < 0 || zz >= g.n0 || yy < 0 || yy >= g.n1 || xx < 0 || xx >= g.n2) continue;
        out.v[out.n++] = g.idx(zz, yy, xx);  // loop order = increasing index
      }
  return out;
}

bool valid(const Grid& g, int conn) {
  if (g.n0 < 1 || g.n1 < 1 || g.n2 < 1) return false;
  if (g.ndim == 2) return conn == 4 || conn == 8;
  if (g.ndim == 3) return conn == 6 || conn == 26;
  return false;
}

// ---------------------------------------------------------------------------------
// O1: separable sampled Gaussian on x/255, r = floor(3 sigma + 0.5), normalised weights,
//     clamp-to-edge; sigma == 0 is the identity (C8).
// ---------------------------------------------------------------------------------
void blur_axis(const Grid& g, std::vector<double>& a, int axis, double sigma) {
  int r = (int)std::floor(3.0 * sigma + 0.5);
  std::vector<double> w(2 * r + 1);
  double s = 0;
  for (int i = -r; i <= r; ++i) { w[i + r] = std::exp(-(double)i * i / (2.0 * sigma * sigma)); s += w[i + r]; }
  for (auto& v : w) v /= s;
  int64_t len = axis == 0 ? g.n0 : axis == 1 ? g.n1 : g.n2;
  std::vector<double> out(a.size());
  for (int64_t z = 0; z < g.n0; ++z)
    for (int64_t y = 0; y < g.n1; ++y)
      for (int64_t x = 0; x < g.n2; ++x) {
        int64_t c = axis == 0 ? z : axis == 1 ? y : x;
        double acc = 0;
        for (int i = -r; i <= r; ++i) {
          int64_t k = std::min<int64_t>(std::max<int64_t>(c + i, 0), len - 1);  // clamp
          int64_t q = axis == 0 ? g.idx(k, y, x) : axis == 1 ? g.idx(z, k, x) : g.idx(z, y, k);
          acc += w[i + r] * a[q];
        }
        out[g.idx(z, y, x)] = acc;
      }
  a.swap(out);
}

// O2: per-axis derivative (numpy.gradient convention, edge_order=1): central difference
//     inside, one-sided at the two ends, 0 for an axis of length 1 (C9).
double deriv(const Grid& g, const std::vector<double>& b, int axis, int64_t z, int64_t y, int64_t x) {
  int64_t len = axis == 0 ? g.n0 : axis == 1 ? g.n1 : g.n2;
  if (len < 2) return 0.0;
  int64_t c = axis == 0 ? z : axis == 1 ? y : x;
  auto at = [&](int64_t k) {
    return axis == 0 ? b[g.idx(k, y, x)] : axis == 1 ? b[g.idx(z, k, x)] : b[g.idx(z, y, k)];
  };
  if (c == 0) return at(1) - at(0);
  if (c == len - 1) return at(len - 1) - at(len - 2);
  return (at(c + 1) - at(c - 1)) / 2.0;
}

}  // namespace

extern "C" {

// Returns 0 on success, 1 on invalid arguments.  Outputs: blur, grad (fp64, may be NULL),
// grad_q (u8, may be NULL): q = min(255, floor(255 g + 0.5)) (C10).
}  // extern "C"

template <class Tin, class Tq>
int gradient_impl(const Tin* img, int ndim, int64_t n0, int64_t n1, int64_t n2, double sigma, double vmax,
                  double* blur_out, double* grad_out, Tq* grad_q) {
  Grid g{ndim, n0, n1, n2};
  if ((ndim != 2 && ndim != 3) || n0 < 1 || n1 < 1 || n2 < 1 || !(sigma >= 0)) return 1;
  int64_t N = g.N();
  std::vector<double> b(N);
  for (int64_t p = 0; p < N; ++p) b[p] = img[p] / vmax;  // x / 255 (C8); x / 65535 for 16-bit images
  if (sigma > 0) {
    if (ndim == 3) blur_axis(g, b, 0, sigma);
    blur_axis(g, b, 1, sigma);
    blur_axis(g, b, 2, sigma);
  }
  for (int64_t z = 0; z < n0; ++z)
    for (int64_t y = 0; y < n1; ++y)
      for (int64_t x = 0; x < n2; ++x) {
        double s = 0;
        for (int axis = (ndim == 3 ? 0 : 1); axis < 3; ++axis) {
          double d = deriv(g, b, axis, z, y, x);
          s += d * d;
        }
        double gm = std::sqrt(s);
        int64_t p = g.idx(z, y, x);
        if (blur_out) blur_out[p] = b[p];
        if (grad_out) grad_out[p] = gm;
        if (grad_q) {
          double q = std::floor(vmax * gm + 0.5);  // C10 (vmax = 255); 65535 for 16 bits
          grad_q[p] = (Tq)(q > vmax ? vmax : q);
        }
      }
  return 0;
}

extern "C" {

int oracle_gradient(const uint8_t* img, int ndim, int64_t n0, int64_t n1, int64_t n2,
                    double sigma, double* blur_out, double* grad_out, uint8_t* grad_q) {
  return gradient_impl(img, ndim, n0, n1, n2, sigma, 255.0, blur_out, grad_out, grad_q);
}

// 16-bit images (NEXT f4): b = G * (img / 65535), q = min(65535, floor(65535 g + 0.5)).
int oracle_gradient_u16(const uint16_t* img, int ndim, int64_t n0, int64_t n1, int64_t n2,
                        double sigma, double* blur_out, double* grad_out, uint16_t* grad_q) {
  return gradient_impl(img, ndim, n0, n1, n2, sigma, 65535.0, blur_out, grad_out, grad_q);
}

// ---------------------------------------------------------------------------------
// O3-O4: the watershed partition.
//   lower(p)  <=> some n in N(p) has I(n) < I(p)                          (Alg.1 l.3)
//   Eq. 1     q = max{ r in N(p) : I(r) = min_{n in N(p)} I(n) }           (C3)
//   plateau   = maximal equal-intensity connected set under conn (singletons included)
//   non-minimal plateau (contains a lower voxel): multi-source BFS inside the plateau from
//     its lower voxels gives d; a voxel with d > 0 points to the MAX-index equal neighbour
//     with distance d-1 (Sync step II semantics, P:194-203 + C5/C6)
//   minimal plateau (no lower voxel) = a regional minimum = a terminal
//   region(p) = the minimal plateau reached by following pointers; label = min voxel index
//     in the region (C7).
// Optional dumps: dist (0 lower, BFS d on non-minimal plateaux, -1 on minimal plateaux),
// ptr (parent; p itself for minimal-plateau voxels), n_regions.
// Returns 0 on success, 1 on invalid arguments.
// ---------------------------------------------------------------------------------
}  // extern "C"

template <class Px>
int watershed_impl(const Px* I, int ndim, int64_t n0, int64_t n1, int64_t n2, int conn,
                   int32_t* labels, int32_t* dist_out, int64_t* ptr_out, int64_t* n_regions) {
  Grid g{ndim, n0, n1, n2};
  if (!valid(g, conn)) return 1;
  int64_t N = g.N();

  // plateaux by sequential flood fill
  std::vector<int64_t> plat(N, -1);
  int64_t n_plat = 0;
  for (int64_t s = 0; s < N; ++s) {
    if (plat[s] >= 0) continue;
    std::deque<int64_t> dq{s};
    plat[s] = n_plat;
    while (!dq.empty()) {
      int64_t p = dq.front(); dq.pop_front();
      for (int64_t q : neighbours(g, conn, p))
        if (plat[q] < 0 && I[q] == I[p]) { plat[q] = n_plat; dq.push_back(q); }
    }
    ++n_plat;
  }

  // lower voxels and Eq. 1
  std::vector<char> lower(N, 0);
  std::vector<int64_t> ptr(N, -1);
  std::vector<char> plat_nonmin(n_plat, 0);
  for (int64_t p = 0; p < N; ++p) {
    auto nb = neighbours(g, conn, p);
    if (nb.empty()) continue;  // single-voxel image: terminal (C4)
    int m = 1 << 16;  // above every u8 / u16 intensity
    for (int64_t q : nb) m = std::min<int>(m, I[q]);
    if (m < I[p]) {
      lower[p] = 1;
      plat_nonmin[plat[p]] = 1;
      int64_t q_eq1 = -1;
      for (int64_t q : nb) if (I[q] == m) q_eq1 = std::max(q_eq1, q);
      ptr[p] = q_eq1;
    }
  }

  // BFS distances on non-minimal plateaux (all plateaux at once: sources never cross
  // plateaux because BFS only follows equal-intensity edges)
  std::vector<int64_t> dist(N, -1);
  std::deque<int64_t> dq;
  for (int64_t p = 0; p < N; ++p) if (lower[p]) { dist[p] = 0; dq.push_back(p); }
  while (!dq.empty()) {
    int64_t p = dq.front(); dq.pop_front();
    for (int64_t q : neighbours(g, conn, p))
      if (dist[q] < 0 && I[q] == I[p]) { dist[q] = dist[p] + 1; dq.push_back(q); }
  }
  for (int64_t p = 0; p < N; ++p) {
    if (dist[p] > 0) {
      int64_t best = -1;
      for (int64_t q : neighbours(g, conn, p))
        if (I[q] == I[p] && dist[q] == dist[p] - 1) best = std::max(best, q);
      ptr[p] = best;
    } else if (dist[p] < 0) {
      ptr[p] = p;  // minimal plateau voxel: terminal
    }
  }

  // follow pointers to the terminal minimal plateau (memoised, iterative)
  std::vector<int64_t> term(N, -1);  // plateau id of the regional minimum reached
  std::vector<int64_t> path;
  for (int64_t s = 0; s < N; ++s) {
    int64_t p = s;
    path.clear();
    while (term[p] < 0 && ptr[p] != p) { path.push_back(p); p = ptr[p]; }
    int64_t t = term[p] >= 0 ? term[p] : plat[p];
    term[p] = t;
    for (int64_t v : path) term[v] = t;
  }
  // canonical label = smallest voxel index of the region
  std::vector<int64_t> minidx(n_plat, INT64_MAX);
  for (int64_t p = 0; p < N; ++p) minidx[term[p]] = std::min(minidx[term[p]], p);
  int64_t R = 0;
  for (int64_t p = 0; p < N; ++p) {
    if (labels) labels[p] = (int32_t)minidx[term[p]];
    if (minidx[term[p]] == p) ++R;
    if (dist_out) dist_out[p] = (int32_t)dist[p];
    if (ptr_out) ptr_out[p] = ptr[p];
  }
  if (n_regions) *n_regions = R;
  return 0;
}

extern "C" {

int oracle_watershed(const uint8_t* I, int ndim, int64_t n0, int64_t n1, int64_t n2, int conn,
                     int32_t* labels, int32_t* dist_out, int64_t* ptr_out, int64_t* n_regions) {
  return watershed_impl(I, ndim, n0, n1, n2, conn, labels, dist_out, ptr_out, n_regions);
}

// The same definition on a 16-bit image (NEXT f4): intensities compare as u16.
int oracle_watershed_u16(const uint16_t* I, int ndim, int64_t n0, int64_t n1, int64_t n2, int conn,
                         int32_t* labels, int32_t* dist_out, int64_t* ptr_out, int64_t* n_regions) {
  return watershed_impl(I, ndim, n0, n1, n2, conn, labels, dist_out, ptr_out, n_regions);
}

// ---------------------------------------------------------------------------------
// O6-O7: the waterfall hierarchy over the region adjacency graph.
//   RAG: for p and q in N(p), q > p, label(p) != label(q): an edge {label(p), label(q)}
//        with height max(I(p), I(q)); per pair keep the MIN height (Alg. 4 l.2-7).
//   K  : strict total order (w asc, max(a,b) desc, min(a,b) desc) on canonical labels (C14).
//   level 0 = labels.  Level k (1..NL-1): every component of level k-1 picks its min-K edge
//        to another component; all picks are merged (min-root union-find on labels, C16);
//        a component with no outgoing edge stays as is (C17).
//   levels[k*N + p] = smallest voxel index of p's level-k region; counts[k] = #regions.
// `labels` must be a canonical watershed labelling.  Returns 0 ok, 1 invalid args.
// ---------------------------------------------------------------------------------
}  // extern "C"

template <class Px>
int waterfall_impl(const int32_t* labels, const Px* I, int ndim, int64_t n0, int64_t n1,
                   int64_t n2, int conn, int NL, int32_t* levels, int64_t* counts) {
  Grid g{ndim, n0, n1, n2};
  if (!valid(g, conn) || NL < 1) return 1;
  int64_t N = g.N();

  std::map<std::pair<int64_t, int64_t>, int> rag;  // (min label, max label) -> min height
  for (int64_t p = 0; p < N; ++p)
    for (int64_t q : neighbours(g, conn, p)) {
      if (q <= p || labels[p] == labels[q]) continue;
      std::pair<int64_t, int64_t> key(std::min(labels[p], labels[q]), std::max(labels[p], labels[q]));
      int h = std::max<int>(I[p], I[q]);
      auto it = rag.find(key);
      if (it == rag.end()) rag[key] = h; else it->second = std::min(it->second, h);
    }
  struct Edge { int w; int64_t a, b; };  // a = min label, b = max label
  std::vector<Edge> edges;
  for (auto& kv : rag) edges.push_back({kv.second, kv.first.first, kv.first.second});
  std::sort(edges.begin(), edges.end(), [](const Edge& e, const Edge& f) {  // K (C14)
    if (e.w != f.w) return e.w < f.w;
    if (e.b != f.b) return e.b > f.b;
    return e.a > f.a;
  });

  // union-find over voxel-index labels (only region representatives are used)
  std::vector<int64_t> parent(N, -1);
  std::vector<int64_t> reps;
  for (int64_t p = 0; p < N; ++p) if (labels[p] == p) { parent[p] = p; reps.push_back(p); }
  auto find = [&](int64_t x) { while (parent[x] != x) x = parent[x]; return x; };

  for (int64_t p = 0; p < N; ++p) levels[p] = labels[p];
  if (counts) counts[0] = (int64_t)reps.size();
  std::vector<int64_t> pick(N, -1);  // per component root: index of its min-K edge
  for (int k = 1; k < NL; ++k) {
    // each component's min-K outgoing edge: the first in K order touching it
    for (int64_t r : reps) pick[r] = -1;
    for (size_t e = 0; e < edges.size(); ++e) {
      int64_t ca = find(edges[e].a), cb = find(edges[e].b);
      if (ca == cb) continue;
      if (pick[ca] < 0) pick[ca] = (int64_t)e;
      if (pick[cb] < 0) pick[cb] = (int64_t)e;
    }
    for (int64_t r : reps) {  // merge along every pick, smaller root wins (C16)
      if (pick[r] < 0) continue;
      int64_t ca = find(edges[pick[r]].a), cb = find(edges[pick[r]].b);
      if (ca == cb) continue;
      if (ca < cb) parent[cb] = ca; else parent[ca] = cb;
    }
    int64_t R = 0;
    for (int64_t r : reps) if (find(r) == r) ++R;
    if (counts) counts[k] = R;
    for (int64_t p = 0; p < N; ++p) levels[(int64_t)k * N + p] = (int32_t)find(labels[p]);
  }
  return 0;
}

extern "C" {

int oracle_waterfall(const int32_t* labels, const uint8_t* I, int ndim, int64_t n0, int64_t n1,
                     int64_t n2, int conn, int NL, int32_t* levels, int64_t* counts) {
  return waterfall_impl<uint8_t>(labels, I, ndim, n0, n1, n2, conn, NL, levels, counts);
}

// O12, the same definition on a 16-bit image (NEXT f4): pass heights max(I(p), I(q))
// compare as u16, so K (C14) orders 16-bit heights first.
int oracle_waterfall_u16(const int32_t* labels, const uint16_t* I, int ndim, int64_t n0, int64_t n1,
                         int64_t n2, int conn, int NL, int32_t* levels, int64_t* counts) {
  return waterfall_impl<uint16_t>(labels, I, ndim, n0, n1, n2, conn, NL, levels, counts);
}

// ---------------------------------------------------------------------------------
// O9: the paper-literal waterfall by image reconstruction (Alg. 4; Alg. 5,
// P:630-656).  Level 0 = labels on the input image I_0 = I.  Level k
// (1..NL-1), from I_{k-1} and L_{k-1}:
//   V  newmin(l) = M, then for every p and q in N(p) with L(q) != L(p):
//        newmin(L(p)) = min(newmin(L(p)), max(I(p), I(q)))          (Alg. 4 l.1-7)
//   VI I_k(p) = max(I_{k-1}(p), newmin(L(p)))                        (Alg. 4 l.8-12)
//   L_k = watershed of I_k (O3-O4: the same definition as level 0)   (Alg. 5 l.4-8)
// M = 255, the upper bound of the u8 greyscale range ("at least the upper bound";
// reading C23).  levels[k*N + p] = L_k(p) (canonical labels); counts[k] = #regions.
// Returns 0 ok, 1 invalid args.
// ---------------------------------------------------------------------------------
int oracle_waterfall_reconstruct(const int32_t* labels, const uint8_t* I, int ndim, int64_t n0, int64_t n1,
                                 int64_t n2, int conn, int NL, int32_t* levels, int64_t* counts) {
  Grid g{ndim, n0, n1, n2};
  if (!valid(g, conn) || NL < 1) return 1;
  const int64_t N = g.N();
  const int M = 255;
  std::vector<uint8_t> img(I, I + N);
  std::vector<int32_t> L(labels, labels + N);
  int64_t R0 = 0;
  for (int64_t p = 0; p < N; ++p) {
    levels[p] = L[p];
    R0 += L[p] == p;
  }
  if (counts) counts[0] = R0;
  std::vector<int> newmin(N);
  for (int k = 1; k < NL; ++k) {
    std::fill(newmin.begin(), newmin.end(), M);  // step V
    for (int64_t p = 0; p < N; ++p)
      for (int64_t q : neighbours(g, conn, p)) {
        if (L[q] == L[p]) continue;
        const int h = std::max<int>(img[p], img[q]);
        if (h < newmin[L[p]]) newmin[L[p]] = h;
      }
    for (int64_t p = 0; p < N; ++p)  // step VI
      if (img[p] < newmin[L[p]]) img[p] = (uint8_t)newmin[L[p]];
    int64_t R = 0;
    if (oracle_watershed(img.data(), ndim, n0, n1, n2, conn, L.data(), nullptr, nullptr, &R) != 0) return 1;
    for (int64_t p = 0; p < N; ++p) levels[(int64_t)k * N + p] = L[p];
    if (counts) counts[k] = R;
  }
  return 0;
}

}  // extern "C"
