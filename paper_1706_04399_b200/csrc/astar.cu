// Voxel A* legs for a tour (graph.py:30-38, 58-66 and
// voxel.py:112-172), host code.  The device builds the cost matrix by
// multi-source shortest paths (k_sssp.cu); the waypoint legs of the N edges
// of the final tour come from this restatement of the reference's A*, which
// reproduces its path choice exactly: heap entries ordered by (f, g, voxel
// index), came-from updated only on a strict improvement, neighbours in the
// reference's NEIGHBOR_STEPS order, the same fp64 expressions for the step
// costs and both heuristics.  Each (start, goal) search is independent, so a
// batch runs on all host cores.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <unistd.h>

#include <algorithm>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "dpso_internal.cuh"

namespace {

int fail(int code, const char* msg) { return dpso::api_fail(code, msg); }

struct Grid {
  const uint8_t* occ;
  int nx, ny, nz;
  double w[3];
  int64_t at(int x, int y, int z) const {
    return ((int64_t)x * ny + y) * nz + z;
  }
};

struct Entry {
  double f, g;
  int x, y, z;
  // std::priority_queue is a max-heap: "a < b" iff a pops after b
  bool operator<(const Entry& o) const {
    if (f != o.f) return f > o.f;
    if (g != o.g) return g > o.g;
    if (x != o.x) return x > o.x;
    if (y != o.y) return y > o.y;
    return z > o.z;
  }
};

// per-thread scratch over the whole grid, reset through a touched list
struct Scratch {
  std::vector<double> gs;
  std::vector<int64_t> came;
  std::vector<uint8_t> closed;
  std::vector<int64_t> touched;
  void ensure(int64_t cells) {
    if ((int64_t)gs.size() != cells) {
      gs.assign(cells, INFINITY);
      came.assign(cells, -1);
      closed.assign(cells, 0);
    }
  }
  void reset() {
    for (int64_t c : touched) {
      gs[c] = INFINITY;
      came[c] = -1;
      closed[c] = 0;
    }
    touched.clear();
  }
};

double heuristic(const Grid& G, int mode, int x, int y, int z, const int* g) {
  const int d[3] = {x - g[0], y - g[1], z - g[2]};
  if (mode == 0) {  // admissible: max_i w_i |d_i|
    double m = G.w[0] * (double)abs(d[0]);
    for (int i = 1; i < 3; ++i) m = std::max(m, G.w[i] * (double)abs(d[i]));
    return m;
  }
  // paper: squared Euclidean distance in voxel units (an int -> float)
  return (double)(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
}

// returns 0 found, 1 blocked; path written into out (x, y, z triples)
int search(const Grid& G, int mode, const int* s, const int* t, Scratch& S,
           std::vector<int32_t>& out, double* cost) {
  out.clear();
  if (s[0] == t[0] && s[1] == t[1] && s[2] == t[2]) {
    out.insert(out.end(), {s[0], s[1], s[2]});
    *cost = 0.0;
    return 0;
  }
  int steps[26][3];
  double sc[26];
  int k = 0;
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b)
      for (int c = -1; c <= 1; ++c) {
        if (!a && !b && !c) continue;
        steps[k][0] = a;
        steps[k][1] = b;
        steps[k][2] = c;
        // a1*alpha*alpha + a2*beta*beta + a3*gamma*gamma, left to right
        sc[k] = G.w[0] * a * a + G.w[1] * b * b + G.w[2] * c * c;
        ++k;
      }
  std::priority_queue<Entry> pq;
  const int64_t si = G.at(s[0], s[1], s[2]);
  S.gs[si] = 0.0;
  S.touched.push_back(si);
  pq.push({heuristic(G, mode, s[0], s[1], s[2], t), 0.0, s[0], s[1], s[2]});
  const int64_t ti = G.at(t[0], t[1], t[2]);
  while (!pq.empty()) {
    const Entry e = pq.top();
    pq.pop();
    const int64_t ci = G.at(e.x, e.y, e.z);
    if (S.closed[ci]) continue;
    if (ci == ti) {
      std::vector<int64_t> rev;
      for (int64_t c = ci; c != si; c = S.came[c]) rev.push_back(c);
      rev.push_back(si);
      for (auto it = rev.rbegin(); it != rev.rend(); ++it) {
        const int64_t c = *it;
        const int z = (int)(c % G.nz), y = (int)((c / G.nz) % G.ny),
                  x = (int)(c / ((int64_t)G.nz * G.ny));
        out.insert(out.end(), {x, y, z});
      }
      *cost = e.g;
      return 0;
    }
    S.closed[ci] = 1;
    for (int q = 0; q < 26; ++q) {
      const int x = e.x + steps[q][0], y = e.y + steps[q][1],
                z = e.z + steps[q][2];
      if (x < 0 || x >= G.nx || y < 0 || y >= G.ny || z < 0 || z >= G.nz)
        continue;
      const int64_t ni = G.at(x, y, z);
      if (G.occ[ni]) continue;
      const double ng = e.g + sc[q];
      if (ng < S.gs[ni]) {
        if (S.gs[ni] == INFINITY) S.touched.push_back(ni);
        S.gs[ni] = ng;
        S.came[ni] = ci;
        pq.push({ng + heuristic(G, mode, x, y, z, t), ng, x, y, z});
      }
    }
  }
  return 1;
}

}  // namespace

extern "C" int dpso_voxel_paths(const uint8_t* host_occ, int32_t nx,
                                int32_t ny, int32_t nz,
                                const double* weights, int32_t mode,
                                const int32_t* pairs, int32_t k,
                                int32_t* out_xyz, int64_t cap_per,
                                int64_t* lens, double* costs) {
  if (!host_occ || !weights || !pairs || !lens || !costs || k < 0 ||
      nx < 1 || ny < 1 || nz < 1 || (mode != 0 && mode != 1) ||
      (cap_per > 0 && !out_xyz))
    return fail(DPSO_EINVAL, "bad arguments");
  Grid G{host_occ, nx, ny, nz, {weights[0], weights[1], weights[2]}};
  for (int i = 0; i < k; ++i)
    for (int e = 0; e < 2; ++e) {
      const int32_t* p = pairs + 6 * i + 3 * e;
      if (p[0] < 0 || p[0] >= nx || p[1] < 0 || p[1] >= ny || p[2] < 0 ||
          p[2] >= nz)
        return fail(DPSO_EINVAL, "voxel index out of the grid");
      if (host_occ[G.at(p[0], p[1], p[2])]) {
        char m[160];
        snprintf(m, sizeof m, "%s voxel (%d, %d, %d) is occupied",
                 e == 0 ? "start" : "goal", p[0], p[1], p[2]);
        return fail(DPSO_EINVAL, m);
      }
    }
  const int64_t cells = (int64_t)nx * ny * nz;
  long hw = sysconf(_SC_NPROCESSORS_ONLN);
  const int nt = (int)std::max(1L, std::min<long>(std::min(hw, 32L), k));
  std::vector<int> status(k, 0);
  auto work = [&](int t) {
    Scratch S;
    S.ensure(cells);
    std::vector<int32_t> path;
    for (int i = t; i < k; i += nt) {
      double c = 0.0;
      const int r = search(G, mode, pairs + 6 * i, pairs + 6 * i + 3, S,
                           path, &c);
      S.reset();
      if (r) {  // blocked: the reference returns None
        lens[i] = 0;
        costs[i] = INFINITY;
        continue;
      }
      const int64_t len = (int64_t)path.size() / 3;
      lens[i] = len;
      costs[i] = c;
      if (len > cap_per) {
        status[i] = 1;
        continue;
      }
      std::copy(path.begin(), path.end(), out_xyz + 3 * cap_per * i);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (int i = 0; i < k; ++i)
    if (status[i])
      return fail(DPSO_EINVAL, "path longer than the output capacity");
  return DPSO_OK;
}
