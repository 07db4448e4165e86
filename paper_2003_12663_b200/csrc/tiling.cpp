// Host (C++) column tiling of the regular sweep ("device column
// order"): the schedule of (column tile, panel) records the assembly kernel
// (csrc/assemble.cu) streams.  Native because it sits on the end-to-end path
// of every assemble() on a fresh mesh.
//
//  1. Recursive coordinate bisection of the collocation points (median split
//     on the longest extent) into tiles of <= max_tile columns.
//  2. Each tile is swept along its longest axis: its columns are numbered in
//     that order (the device column order is tile after tile).
//  3. Records: one per (panel, tile owning >= 1 of its corners); a record
//     contributes to its owned corners only.  Sorted by (first owned local
//     column, panel).
//  4. Stages of GROUP records (one bulk copy each), first-fit in record
//     order: a record joins the oldest open stage whose first record's first
//     owned column is within `band` of its last owned column and whose owned
//     corners are disjoint from its own, else opens a new stage; stages are
//     emitted in creation order, short ones padded with dummy records (-1).
//     Disjoint owned corners let the kernel update its window for a whole
//     stage without read-after-write chains.
//  5. A tile whose own records span more than `band` columns, or whose
//     stages pad more than 1/8 of their slots, is halved across its sweep
//     direction (second-longest axis) and the pass repeats.
//
// Everything is deterministic (ties broken by index).
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

struct Tiling {
  std::vector<int> perm;          // device column -> original column
  std::vector<int> col0, width;   // per tile
  std::vector<long long> ptr;     // per tile: record offsets (n_tiles + 1)
  std::vector<int> ent_tri;       // per record: panel (-1: dummy)
  std::vector<int> ent_meta;      // per record: mfirst, l0, l1, l2, flags (l = owned local column or -1)
  int band = 0;
  long long real = 0;             // non-dummy records
};

using Pts = const double*;

int longest_axis(Pts p, const std::vector<int>& idx, int rank = 0) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int v : idx)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], p[3 * (size_t)v + d]);
      hi[d] = std::max(hi[d], p[3 * (size_t)v + d]);
    }
  std::array<int, 3> ax = {0, 1, 2};
  // extents descending, ties by axis index
  std::stable_sort(ax.begin(), ax.end(), [&](int a, int b) { return hi[a] - lo[a] > hi[b] - lo[b]; });
  return ax[rank];
}

// stable sort along axis ax: ties (structured grids share coordinates)
// keep the order of the previous split or sweep, which keeps equal-coordinate
// rows geometrically coherent
void sort_along(Pts p, std::vector<int>& idx, int ax) {
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int a, int b) { return p[3 * (size_t)a + ax] < p[3 * (size_t)b + ax]; });
}

void rcb(Pts p, std::vector<int> idx, int max_tile, std::vector<std::vector<int>>& out) {
  std::vector<std::vector<int>> stack;
  stack.push_back(std::move(idx));
  while (!stack.empty()) {
    std::vector<int> cur = std::move(stack.back());
    stack.pop_back();
    if ((int)cur.size() <= max_tile) {
      out.push_back(std::move(cur));
      continue;
    }
    sort_along(p, cur, longest_axis(p, cur));
    const size_t h = cur.size() / 2;
    std::vector<int> a(cur.begin(), cur.begin() + h), b(cur.begin() + h, cur.end());
    stack.push_back(std::move(b));  // second half pushed first: tiles come out in sweep order
    stack.push_back(std::move(a));
  }
}

struct Rec {
  int tri, mfirst, mlast, l[3], flags;
};

struct Done {  // one finished tile
  std::vector<int> cols;      // device order
  std::vector<int> ent_tri;   // records (-1: dummy)
  std::vector<int> ent_meta;  // 5 per record
  int band = 0;
  long long real = 0;
};

struct Ctx {
  Pts p;
  const int* tri_cols;
  std::vector<int> star_ptr, star_tri;  // vertex -> panels (CSR)
  std::vector<int> tile_of, local;      // scratch, valid for the tile being processed
  std::vector<int> seen;                // panel -> last tile stamp
  int stamp = 0;
  int band, group;
};

// Records and stages of one tile; false if the tile must be split (a record
// spans more than `band` columns, or its stages pad more than 1/8 of slots).
bool build_tile(Ctx& C, std::vector<int>& cols, Done& out) {
  sort_along(C.p, cols, longest_axis(C.p, cols));
  const int k = ++C.stamp;
  for (int i = 0; i < (int)cols.size(); ++i) {
    C.tile_of[cols[i]] = k;
    C.local[cols[i]] = i;
  }
  std::vector<Rec> R;
  for (int v : cols)
    for (int s = C.star_ptr[v]; s < C.star_ptr[v + 1]; ++s) {
      const int t = C.star_tri[s];
      if (C.seen[t] == k) continue;
      C.seen[t] = k;
      const int* c = C.tri_cols + 3 * (size_t)t;
      Rec r{t, 1 << 30, -1, {-1, -1, -1}, C.tile_of[c[0]] == k ? 1 : 0};
      for (int i = 0; i < 3; ++i)
        if (C.tile_of[c[i]] == k) {
          r.l[i] = C.local[c[i]];
          r.mfirst = std::min(r.mfirst, r.l[i]);
          r.mlast = std::max(r.mlast, r.l[i]);
        }
      if (r.mlast - r.mfirst > C.band) return false;
      R.push_back(r);
    }
  std::sort(R.begin(), R.end(), [](const Rec& a, const Rec& b) {
    return a.mfirst < b.mfirst || (a.mfirst == b.mfirst && a.tri < b.tri);
  });
  // stages, first-fit in record order: a record joins the oldest open stage
  // it fits (within band of the stage's first record, owned corners
  // disjoint), else opens a new one; stages are emitted in creation order,
  // so stage starts never decrease and every record of a later stage has
  // its first owned column >= this stage's start (the kernel's flush rule)
  const int band = C.band, group = C.group;
  std::vector<std::vector<int>> stages;
  std::vector<int> open;  // indices into stages, creation order
  for (int i = 0; i < (int)R.size(); ++i) {
    const Rec& r = R[i];
    while (!open.empty() && R[stages[open.front()][0]].mfirst + band < r.mfirst) open.erase(open.begin());
    bool placed = false;
    for (size_t o = 0; o < open.size() && !placed; ++o) {
      std::vector<int>& g = stages[open[o]];
      if (r.mlast > R[g[0]].mfirst + band) continue;
      bool clash = false;
      for (int gi : g)
        for (int x = 0; x < 3 && !clash; ++x)
          for (int y = 0; y < 3 && !clash; ++y) clash = R[gi].l[x] >= 0 && R[gi].l[x] == r.l[y];
      if (clash) continue;
      g.push_back(i);
      if ((int)g.size() == group) open.erase(open.begin() + o);
      placed = true;
    }
    if (!placed) {
      stages.push_back({i});
      if (group > 1) open.push_back((int)stages.size() - 1);
    }
  }
  const size_t slots = (size_t)group * stages.size();
  if (R.size() > 64 && 8 * (slots - R.size()) > slots && cols.size() > 1) return false;
  out.cols = cols;
  for (const auto& g : stages) {
    const Rec& r0 = R[g[0]];
    for (int gi : g) {
      const Rec& r = R[gi];
      out.ent_tri.push_back(r.tri);
      out.ent_meta.insert(out.ent_meta.end(), {r.mfirst, r.l[0], r.l[1], r.l[2], r.flags});
      out.band = std::max(out.band, r.mlast - r0.mfirst);
      ++out.real;
    }
    for (int d = (int)g.size(); d < group; ++d) {  // dummy: no owned corner, not primary
      out.ent_tri.push_back(-1);
      out.ent_meta.insert(out.ent_meta.end(), {r0.mfirst, -1, -1, -1, 0});
    }
  }
  return true;
}

// depth-first: a tile that must be split is replaced by its two halves
// (across the sweep direction: the tile stays a strip), in place
bool process(Ctx& C, std::vector<int> cols, std::vector<Done>& out, int depth) {
  Done d;
  if (build_tile(C, cols, d)) {
    out.push_back(std::move(d));
    return true;
  }
  if (cols.size() <= 1 || depth > 48) return false;  // pathological mesh: band not bounded
  sort_along(C.p, cols, longest_axis(C.p, cols, 1));
  const size_t h = cols.size() / 2;
  std::vector<int> a(cols.begin(), cols.begin() + h), b(cols.begin() + h, cols.end());
  return process(C, std::move(a), out, depth + 1) && process(C, std::move(b), out, depth + 1);
}

}  // namespace

extern "C" {

// Returns 0 on success; *handle owns the result until hvb_tiling_free.
// sizes[0..3] = n_tiles, n_records (incl. dummies), band, real records.
int hvb_tiling_build(const double* points, int n, const int* tri_cols, int nt, int max_tile, int band, int group,
                     long long* sizes, void** handle) {
  if (!points || !tri_cols || !sizes || !handle || n <= 0 || nt < 0 || max_tile < 1 || band < 0 || group < 1)
    return 1;
  for (long long i = 0; i < 3ll * nt; ++i)
    if (tri_cols[i] < 0 || tri_cols[i] >= n) return 1;
  Ctx C;
  C.p = points;
  C.tri_cols = tri_cols;
  C.band = band;
  C.group = group;
  C.star_ptr.assign(n + 1, 0);
  for (long long i = 0; i < 3ll * nt; ++i) ++C.star_ptr[tri_cols[i] + 1];
  for (int v = 0; v < n; ++v) C.star_ptr[v + 1] += C.star_ptr[v];
  C.star_tri.resize(3 * (size_t)nt);
  {
    std::vector<int> fill(C.star_ptr.begin(), C.star_ptr.end() - 1);
    for (int t = 0; t < nt; ++t)
      for (int j = 0; j < 3; ++j) C.star_tri[fill[tri_cols[3 * (size_t)t + j]]++] = t;
  }
  std::vector<int> all(n);
  std::iota(all.begin(), all.end(), 0);
  std::vector<std::vector<int>> tiles;
  rcb(points, all, max_tile, tiles);
  // top-level tiles are independent: one worker thread per tile (each with
  // its own scratch), results concatenated in tile order
  const int nw = (int)std::min<size_t>(tiles.size(), std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  std::vector<std::vector<Done>> parts(tiles.size());
  std::vector<char> ok(tiles.size(), 1);
  std::atomic<size_t> next{0};
  auto work = [&]() {
    Ctx W = C;
    W.tile_of.assign(n, 0);
    W.local.assign(n, 0);
    W.seen.assign(nt, 0);
    for (size_t i; (i = next.fetch_add(1)) < tiles.size();) ok[i] = process(W, std::move(tiles[i]), parts[i], 0);
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < nw; ++w) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  std::vector<Done> done;
  for (size_t i = 0; i < tiles.size(); ++i) {
    if (!ok[i]) return 2;
    for (auto& d : parts[i]) done.push_back(std::move(d));
  }
  Tiling* T = new Tiling();
  T->ptr.assign(1, 0);
  int c0 = 0;
  for (auto& d : done) {
    T->perm.insert(T->perm.end(), d.cols.begin(), d.cols.end());
    T->col0.push_back(c0);
    T->width.push_back((int)d.cols.size());
    c0 += (int)d.cols.size();
    T->ent_tri.insert(T->ent_tri.end(), d.ent_tri.begin(), d.ent_tri.end());
    T->ent_meta.insert(T->ent_meta.end(), d.ent_meta.begin(), d.ent_meta.end());
    T->ptr.push_back((long long)T->ent_tri.size());
    T->band = std::max(T->band, d.band);
    T->real += d.real;
  }
  sizes[0] = (long long)done.size();
  sizes[1] = (long long)T->ent_tri.size();
  sizes[2] = T->band;
  sizes[3] = T->real;
  *handle = T;
  return 0;
}

int hvb_tiling_fetch(void* handle, int* perm, int* tile_col0, int* tile_width, long long* tile_ptr, int* ent_tri,
                     int* ent_meta) {
  if (!handle) return 1;
  const Tiling* T = static_cast<const Tiling*>(handle);
  std::memcpy(perm, T->perm.data(), T->perm.size() * sizeof(int));
  std::memcpy(tile_col0, T->col0.data(), T->col0.size() * sizeof(int));
  std::memcpy(tile_width, T->width.data(), T->width.size() * sizeof(int));
  std::memcpy(tile_ptr, T->ptr.data(), T->ptr.size() * sizeof(long long));
  std::memcpy(ent_tri, T->ent_tri.data(), T->ent_tri.size() * sizeof(int));
  std::memcpy(ent_meta, T->ent_meta.data(), T->ent_meta.size() * sizeof(int));
  return 0;
}

int hvb_tiling_free(void* handle) {
  delete static_cast<Tiling*>(handle);
  return 0;
}

}  // extern "C"
