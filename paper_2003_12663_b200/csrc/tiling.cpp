// Host (C++) column tiling of the regular sweep ("device column
// order"): the schedule of (column tile, panel) records the assembly kernel
// (csrc/assemble.cu) streams.  Native because it sits on the end-to-end path
// of every assemble() on a fresh mesh.
//
//  1. Recursive coordinate bisection of the collocation points (median split
//     on the longest extent) into tiles of <= max_tile columns.  A tile OWNS
//     its columns; each tile is swept along its longest axis and its owned
//     columns are numbered in that order (the device column order is tile
//     after tile).
//  2. Records: ONE per panel, in its primary tile = the lowest-numbered tile
//     owning one of its corners, so no panel is evaluated twice.  A tile's
//     LOCAL columns are its owned columns plus its "halo": corners of its
//     panels owned by later tiles.  Local columns are numbered along the
//     sweep axis; records sorted by (first local column, panel).
//  3. Stages of GROUP records (one bulk copy each), first-fit in record
//     order: a record joins the oldest open stage whose first record's first
//     local column is within `band` of its last local column and whose
//     corners are disjoint from its own, else opens a new stage; stages are
//     emitted in creation order, short ones padded with dummy records (-1).
//     Disjoint corners let the kernel update its window for a whole stage
//     without read-after-write chains.
//  4. A tile whose records span more than `band` local columns, or whose
//     stages pad more than 1/8 of their slots, is halved across its sweep
//     direction (second-longest axis); the halves are built in the next
//     pass (halving keeps the order of the other tiles, so their primaries
//     and builds stand).  Before any build, tiles are halved while the span
//     over their owned columns alone exceeds the band (a cheap lower bound).
//  5. Halo exchange through slots of raw partial sums (n_rows doubles
//     each): a producing tile writes its sums of a halo column into the
//     copy's slot; the owning (later) tile writes its own sums of that
//     "receiving" column into a partial slot instead of A; the last CTA of
//     the owner and its producers (same rows) to finish adds partial +
//     copies (producer order) and writes the entry, so each entry is summed
//     in a fixed order and no CTA waits.  Receiving columns are numbered
//     last within their tile, so those writes are contiguous runs of A.
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
  std::vector<int> col0, width;   // per tile: owned device columns
  std::vector<long long> ptr;     // per tile: record offsets (n_tiles + 1)
  std::vector<int> ent_tri;       // per record: panel (-1: dummy)
  std::vector<int> ent_meta;      // per record: mfirst, l0, l1, l2, flags (l = local column, -1 dummy)
  std::vector<int> lptr;          // per tile: local column offsets (n_tiles + 1)
  std::vector<int> lcol;          // per local column: device column, or ~slot (halo copy / partial)
  std::vector<int> xptr;          // per tile: exchange entry offsets (n_tiles + 1)
  std::vector<int> xent;          // per exchange entry: slot, device column, first, last
  std::vector<int> pptr;          // per tile: producer offsets (n_tiles + 1)
  std::vector<int> prods;         // per tile: distinct producer tiles, ascending
  std::vector<int> cptr;          // per tile: consumer offsets (n_tiles + 1)
  std::vector<int> cons;          // per tile: distinct consumer tiles, ascending
  int band = 0;
  long long real = 0;             // non-dummy records
  int n_halo = 0, n_slots = 0;
};

using Pts = const double*;

// Global order of the columns along each axis: (x_a, x_a+1, x_a+2, index)
// lexicographic on the coordinates rounded to float -- gr[a][v] is column
// v's position.  A tile keeps its
// columns sorted along all three axes, so cutting it is a linear stable
// partition and no tile is ever sorted again.
// stable LSD radix sort of idx by coordinate ax rounded to float (the
// order-preserving 32-bit image; two 16-bit digits, a digit shared by all
// keys skipped; -0 == +0)
void radix_sort_along(Pts p, std::vector<int>& idx, int ax) {
  const size_t m = idx.size();
  std::vector<uint32_t> key(m), key2(m);
  std::vector<int> idx2(m);
  for (size_t i = 0; i < m; ++i) {
    float x = (float)p[3 * (size_t)idx[i] + ax];
    if (x == 0.0f) x = 0.0f;
    uint32_t b;
    std::memcpy(&b, &x, 4);
    key[i] = (b >> 31) ? ~b : (b | (1u << 31));
  }
  constexpr int DIG = 16, NB = 1 << DIG;
  std::vector<uint32_t> cnt(NB);
  for (int sh = 0; sh < 32; sh += DIG) {
    std::fill(cnt.begin(), cnt.end(), 0);
    for (size_t i = 0; i < m; ++i) ++cnt[(key[i] >> sh) & (NB - 1)];
    if (*std::max_element(cnt.begin(), cnt.end()) == m) continue;  // one digit value: order unchanged
    uint32_t run = 0;
    for (int d = 0; d < NB; ++d) {
      const uint32_t c = cnt[d];
      cnt[d] = run;
      run += c;
    }
    for (size_t i = 0; i < m; ++i) {
      const uint32_t o = cnt[(key[i] >> sh) & (NB - 1)]++;
      key2[o] = key[i];
      idx2[o] = idx[i];
    }
    key.swap(key2);
    idx.swap(idx2);
  }
}

struct Order {
  std::array<std::vector<int>, 3> gr;
};

struct Tile {
  std::array<std::vector<int>, 3> by;  // columns in global order along each axis
  size_t size() const { return by[0].size(); }
};

// axes by extent descending (ties by axis index): rank 0 = the sweep axis
int longest_axis(Pts p, const Tile& t, int rank = 0) {
  double ext[3];
  for (int d = 0; d < 3; ++d)
    ext[d] = t.size() ? p[3 * (size_t)t.by[d].back() + d] - p[3 * (size_t)t.by[d].front() + d] : 0.0;
  std::array<int, 3> ax = {0, 1, 2};
  std::stable_sort(ax.begin(), ax.end(), [&](int a, int b) { return ext[a] > ext[b]; });
  return ax[rank];
}

// halve t along axis a (first half: the lower positions along a)
void halve(const Tile& t, int a, Tile& lo, Tile& hi, std::vector<int>& mark, int& stamp) {
  const size_t h = t.size() / 2;
  const int st = ++stamp;
  lo.by[a].assign(t.by[a].begin(), t.by[a].begin() + h);
  hi.by[a].assign(t.by[a].begin() + h, t.by[a].end());
  for (int v : lo.by[a]) mark[v] = st;
  for (int d = 0; d < 3; ++d) {
    if (d == a) continue;
    lo.by[d].clear();
    hi.by[d].clear();
    lo.by[d].reserve(h);
    hi.by[d].reserve(t.size() - h);
    for (int v : t.by[d]) (mark[v] == st ? lo : hi).by[d].push_back(v);
  }
}

void rcb(Pts p, Tile all, int max_tile, std::vector<Tile>& out, std::vector<int>& mark, int& stamp) {
  std::vector<Tile> stack;
  stack.push_back(std::move(all));
  while (!stack.empty()) {
    Tile cur = std::move(stack.back());
    stack.pop_back();
    if ((int)cur.size() <= max_tile) {
      out.push_back(std::move(cur));
      continue;
    }
    Tile a, b;
    halve(cur, longest_axis(p, cur), a, b, mark, stamp);
    stack.push_back(std::move(b));  // second half pushed first: tiles come out in sweep order
    stack.push_back(std::move(a));
  }
}

struct Rec {
  int tri, mfirst, mlast, l[3];
};

struct Done {  // one finished tile
  std::vector<int> lcols;     // local columns (original ids), window order
  std::vector<int> ent_tri;   // records (-1: dummy)
  std::vector<int> ent_meta;  // 5 per record
  int band = 0;
  long long real = 0;
};

struct Ctx {
  Pts p;
  const Order* ord;
  const int* tri_cols;
  const std::vector<int>* star_ptr;
  const std::vector<int>* star_tri;
  const std::vector<int>* home;   // column -> owning tile (current numbering)
  std::vector<int> local, lstamp;  // scratch, valid for the tile being processed
  std::vector<int> seen;           // panel -> last stamp
  int stamp = 0;
  int band, group;
};

// Records and stages of tile k (owned columns `cols`, sorted in place along
// the sweep axis); false if the tile must be split (a record spans more
// than `band` local columns, or its stages pad more than 1/8 of slots).
bool build_tile(Ctx& C, int k, const Tile& tile, Done& out) {
  const int ax = longest_axis(C.p, tile);
  const std::vector<int>& cols = tile.by[ax];
  const std::vector<int>& g = C.ord->gr[ax];
  const std::vector<int>& home = *C.home;
  const int st = ++C.stamp;
  std::vector<int> tris, halo;
  for (int v : cols) C.lstamp[v] = st;
  for (int v : cols)
    for (int s = (*C.star_ptr)[v]; s < (*C.star_ptr)[v + 1]; ++s) {
      const int t = (*C.star_tri)[s];
      if (C.seen[t] == st) continue;
      C.seen[t] = st;
      const int* c = C.tri_cols + 3 * (size_t)t;
      if (std::min(home[c[0]], std::min(home[c[1]], home[c[2]])) != k) continue;  // primary elsewhere
      tris.push_back(t);
      for (int i = 0; i < 3; ++i)
        if (C.lstamp[c[i]] != st) {  // halo: owned by a later tile
          C.lstamp[c[i]] = st;
          halo.push_back(c[i]);
        }
    }
  // local columns: owned and halo merged in the global order along ax
  std::sort(halo.begin(), halo.end(), [&](int a, int b) { return g[a] < g[b]; });
  std::vector<int> lcols(cols.size() + halo.size());
  std::merge(cols.begin(), cols.end(), halo.begin(), halo.end(), lcols.begin(),
             [&](int a, int b) { return g[a] < g[b]; });
  for (int i = 0; i < (int)lcols.size(); ++i) C.local[lcols[i]] = i;
  std::sort(tris.begin(), tris.end());
  std::vector<Rec> R;
  R.reserve(tris.size());
  for (int t : tris) {
    const int* c = C.tri_cols + 3 * (size_t)t;
    Rec r{t, 1 << 30, -1, {-1, -1, -1}};
    for (int i = 0; i < 3; ++i) {
      r.l[i] = C.local[c[i]];
      r.mfirst = std::min(r.mfirst, r.l[i]);
      r.mlast = std::max(r.mlast, r.l[i]);
    }
    if (r.mlast - r.mfirst > C.band) return false;
    R.push_back(r);
  }
  std::stable_sort(R.begin(), R.end(), [](const Rec& a, const Rec& b) { return a.mfirst < b.mfirst; });
  // stages, first-fit in record order: a record joins the oldest open stage
  // it fits (within band of the stage's first record, corners disjoint),
  // else opens a new one; stages are emitted in creation order, so stage
  // starts never decrease and every record of a later stage has its first
  // local column >= this stage's start (the kernel's flush rule)
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
          for (int y = 0; y < 3 && !clash; ++y) clash = R[gi].l[x] == r.l[y];
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
  out.lcols = lcols;
  for (const auto& g : stages) {
    const Rec& r0 = R[g[0]];
    for (int gi : g) {
      const Rec& r = R[gi];
      out.ent_tri.push_back(r.tri);
      out.ent_meta.insert(out.ent_meta.end(), {r.mfirst, r.l[0], r.l[1], r.l[2], 1});
      out.band = std::max(out.band, r.mlast - r0.mfirst);
      ++out.real;
    }
    for (int d = (int)g.size(); d < group; ++d) {  // dummy: no corner (window dump slot), never emits
      out.ent_tri.push_back(-1);
      out.ent_meta.insert(out.ent_meta.end(), {r0.mfirst, -1, -1, -1, 0});
    }
  }
  return true;
}

// Widest span of the tile's panels over its owned columns numbered along
// its longest axis (halo corners ignored: a lower bound of the span the
// build checks against the band).
int owned_span(Pts p, const int* tri_cols, const std::vector<int>& star_ptr, const std::vector<int>& star_tri,
               std::vector<int>& rank, const Tile& tile) {
  const std::vector<int>& cols = tile.by[longest_axis(p, tile)];
  for (int i = 0; i < (int)cols.size(); ++i) rank[cols[i]] = i + 1;
  int span = 0;
  for (int v : cols)
    for (int s = star_ptr[v]; s < star_ptr[v + 1]; ++s) {
      const int* c = tri_cols + 3 * (size_t)star_tri[s];
      int lo = 1 << 30, hi = -1;
      for (int i = 0; i < 3; ++i)
        if (rank[c[i]] > 0) {
          lo = std::min(lo, rank[c[i]]);
          hi = std::max(hi, rank[c[i]]);
        }
      span = std::max(span, hi - lo);
    }
  for (int v : cols) rank[v] = 0;
  return span;
}

}  // namespace

extern "C" {

// Returns 0 on success; *handle owns the result until hvb_tiling_free.
// sizes[0..8] = n_tiles, n_records (incl. dummies), band, real records,
// local columns (summed over tiles), exchange entries, slots (halo copies
// + partials), halo copies, producer entries.
int hvb_tiling_build(const double* points, int n, const int* tri_cols, int nt, int max_tile, int band, int group,
                     long long* sizes, void** handle) {
  if (!points || !tri_cols || !sizes || !handle || n <= 0 || nt < 0 || max_tile < 1 || band < 0 || group < 1)
    return 1;
  for (long long i = 0; i < 3ll * nt; ++i)
    if (tri_cols[i] < 0 || tri_cols[i] >= n) return 1;
  std::vector<int> star_ptr(n + 1, 0), star_tri(3 * (size_t)nt);
  for (long long i = 0; i < 3ll * nt; ++i) ++star_ptr[tri_cols[i] + 1];
  for (int v = 0; v < n; ++v) star_ptr[v + 1] += star_ptr[v];
  {
    std::vector<int> fill(star_ptr.begin(), star_ptr.end() - 1);
    for (int t = 0; t < nt; ++t)
      for (int j = 0; j < 3; ++j) star_tri[fill[tri_cols[3 * (size_t)t + j]]++] = t;
  }
  const int nw = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  // global order along each axis (three sorts in parallel)
  Order ord;
  Tile all;
  {
    std::vector<std::thread> th;
    for (int a = 0; a < 3; ++a)
      th.emplace_back([&, a]() {
        std::vector<int>& o = all.by[a];
        o.resize(n);
        std::iota(o.begin(), o.end(), 0);
        for (int r = 2; r >= 0; --r) radix_sort_along(points, o, (a + r) % 3);  // (x_a, x_a+1, x_a+2) lexicographic
        ord.gr[a].resize(n);
        for (int i = 0; i < n; ++i) ord.gr[a][o[i]] = i;
      });
    for (auto& t : th) t.join();
  }
  std::vector<int> mark(n, 0);
  int stamp = 0;
  std::vector<Tile> tiles;
  rcb(points, std::move(all), max_tile, tiles, mark, stamp);
  // Cut tile k across its sweep direction (in place in the tile list).
  auto cut = [&](std::vector<Tile>& out, Tile& t) {
    Tile a, b;
    halve(t, longest_axis(points, t, 1), a, b, mark, stamp);
    out.push_back(std::move(a));
    out.push_back(std::move(b));
  };
  // presplit, level by level in parallel: a tile whose owned span exceeds
  // the band is halved across its sweep direction, and the halves checked
  {
    std::vector<std::vector<int>> ranks(nw);
    std::vector<int> span(tiles.size(), 0);
    std::vector<char> checked(tiles.size(), 0);
    for (int level = 0; level < 48; ++level) {
      std::vector<size_t> todo;
      for (size_t k = 0; k < tiles.size(); ++k)
        if (!checked[k]) todo.push_back(k);
      if (todo.empty()) break;
      std::atomic<size_t> next{0};
      auto work = [&](int w) {
        std::vector<int>& rank = ranks[w];
        if (rank.empty()) rank.assign(n, 0);
        for (size_t i; (i = next.fetch_add(1)) < todo.size();) {
          const size_t k = todo[i];
          span[k] = tiles[k].size() <= 1 ? 0 : owned_span(points, tri_cols, star_ptr, star_tri, rank, tiles[k]);
          checked[k] = 1;
        }
      };
      std::vector<std::thread> pool;
      for (int w = 1; w < std::min<int>(nw, (int)todo.size()); ++w) pool.emplace_back(work, w);
      work(0);
      for (auto& th : pool) th.join();
      std::vector<Tile> nt_tiles;
      std::vector<int> nt_span;
      std::vector<char> nt_checked;
      for (size_t k = 0; k < tiles.size(); ++k) {
        if (span[k] <= band) {
          nt_tiles.push_back(std::move(tiles[k]));
          nt_span.push_back(span[k]);
          nt_checked.push_back(1);
          continue;
        }
        cut(nt_tiles, tiles[k]);
        nt_span.insert(nt_span.end(), {0, 0});
        nt_checked.insert(nt_checked.end(), {0, 0});
      }
      tiles.swap(nt_tiles);
      span.swap(nt_span);
      checked.swap(nt_checked);
    }
  }
  std::vector<int> home(n);
  std::vector<Done> done(tiles.size());
  std::vector<char> built(tiles.size(), 0), ok(tiles.size(), 0);
  std::vector<Ctx> ctx(nw);
  for (Ctx& W : ctx) {
    W.p = points;
    W.ord = &ord;
    W.tri_cols = tri_cols;
    W.star_ptr = &star_ptr;
    W.star_tri = &star_tri;
    W.home = &home;
    W.band = band;
    W.group = group;
  }
  // Passes: build the tiles not built yet, halve the failing ones in place.
  // Halving tile s keeps the relative order of all others, so a panel not
  // touching s keeps its primary tile and every other tile's build stands;
  // only the two halves are (re)built in the next pass.
  for (int pass = 0;; ++pass) {
    if (pass > 64) return 2;  // pathological mesh: band not bounded
    for (size_t k = 0; k < tiles.size(); ++k)
      for (int v : tiles[k].by[0]) home[v] = (int)k;
    std::vector<size_t> todo;
    for (size_t k = 0; k < tiles.size(); ++k)
      if (!built[k]) todo.push_back(k);
    std::atomic<size_t> next{0};
    auto work = [&](int w) {
      Ctx& W = ctx[w];
      if (W.local.empty()) {
        W.local.assign(n, 0);
        W.lstamp.assign(n, 0);
        W.seen.assign(nt, 0);
      }
      for (size_t i; (i = next.fetch_add(1)) < todo.size();) {
        const size_t k = todo[i];
        done[k] = Done();
        ok[k] = build_tile(W, (int)k, tiles[k], done[k]);
        built[k] = 1;
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < std::min<int>(nw, (int)todo.size()); ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& th : pool) th.join();
    if (std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; })) break;
    std::vector<Tile> nt_tiles;
    std::vector<Done> nt_done;
    std::vector<char> nt_built, nt_ok;
    for (size_t k = 0; k < tiles.size(); ++k) {
      if (ok[k]) {
        nt_tiles.push_back(std::move(tiles[k]));
        nt_done.push_back(std::move(done[k]));
        nt_built.push_back(1);
        nt_ok.push_back(1);
        continue;
      }
      if (tiles[k].size() <= 1) return 2;
      cut(nt_tiles, tiles[k]);
      for (int i = 0; i < 2; ++i) {
        nt_done.emplace_back();
        nt_built.push_back(0);
        nt_ok.push_back(0);
      }
    }
    tiles.swap(nt_tiles);
    done.swap(nt_done);
    built.swap(nt_built);
    ok.swap(nt_ok);
  }
  // each tile's owned columns in sweep order
  std::vector<std::vector<int>> owned(tiles.size());
  for (size_t k = 0; k < tiles.size(); ++k) owned[k] = tiles[k].by[longest_axis(points, tiles[k])];
  Tiling* T = new Tiling();
  // halo slots in tile order; hl[v] = (slot, producer) of every halo copy of
  // column v, producers ascending
  std::vector<std::vector<std::array<int, 2>>> hl(n);
  for (size_t k = 0; k < tiles.size(); ++k)
    for (int v : done[k].lcols)
      if (home[v] != (int)k) hl[v].push_back({T->n_halo++, (int)k});
  // device columns: per tile its owned columns without halo copies (sweep
  // order), then the receiving ones (sweep order); a receiving column gets a
  // "partial" slot (after the halo slots) for its own sums
  std::vector<int> dev(n), pslot(n, -1);
  int n_slots = T->n_halo;
  T->ptr.assign(1, 0);
  T->lptr.assign(1, 0);
  T->xptr.assign(1, 0);
  T->pptr.assign(1, 0);
  T->perm.reserve(n);
  int c0 = 0;
  for (size_t k = 0; k < tiles.size(); ++k) {
    T->col0.push_back(c0);
    for (int pass2 = 0; pass2 < 2; ++pass2)
      for (int v : owned[k])
        if (hl[v].empty() == (pass2 == 0)) {
          dev[v] = c0++;
          T->perm.push_back(v);
          if (pass2) pslot[v] = n_slots++;
        }
    T->width.push_back(c0 - T->col0.back());
    const Done& d = done[k];
    T->ptr.push_back(T->ptr.back() + (long long)d.ent_tri.size());
    T->band = std::max(T->band, d.band);
    T->real += d.real;
  }
  // the records of all tiles, copied in parallel to their offsets
  T->ent_tri.resize(T->ptr.back());
  T->ent_meta.resize(5 * T->ptr.back());
  {
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t k; (k = next.fetch_add(1)) < tiles.size();) {
        std::copy(done[k].ent_tri.begin(), done[k].ent_tri.end(), T->ent_tri.begin() + T->ptr[k]);
        std::copy(done[k].ent_meta.begin(), done[k].ent_meta.end(), T->ent_meta.begin() + 5 * T->ptr[k]);
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < std::min<int>(nw, (int)tiles.size()); ++w) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  }
  for (size_t k = 0; k < tiles.size(); ++k) {
    // local columns: device column, or ~slot (halo copy / partial)
    for (int v : done[k].lcols) {
      if (home[v] == (int)k) {
        T->lcol.push_back(pslot[v] < 0 ? dev[v] : ~pslot[v]);
      } else {
        int slot = -1;
        for (const auto& h : hl[v])
          if (h[1] == (int)k) slot = h[0];
        T->lcol.push_back(~slot);
      }
    }
    T->lptr.push_back((int)T->lcol.size());
    // exchange entries of the receiving columns, device order: partial
    // first, then the halo copies by producer; and the distinct producers
    std::vector<int> prods;
    for (int v : owned[k]) {
      if (hl[v].empty()) continue;
      T->xent.insert(T->xent.end(), {pslot[v], dev[v], 1, 0});
      for (size_t i = 0; i < hl[v].size(); ++i) {
        T->xent.insert(T->xent.end(), {hl[v][i][0], dev[v], 0, i + 1 == hl[v].size() ? 1 : 0});
        prods.push_back(hl[v][i][1]);
      }
    }
    std::sort(prods.begin(), prods.end());
    prods.erase(std::unique(prods.begin(), prods.end()), prods.end());
    T->prods.insert(T->prods.end(), prods.begin(), prods.end());
    T->pptr.push_back((int)T->prods.size());
    T->xptr.push_back((int)(T->xent.size() / 4));
  }
  // consumers: the transpose of the producer lists
  {
    std::vector<std::vector<int>> cl(tiles.size());
    for (size_t k = 0; k < tiles.size(); ++k)
      for (int i = T->pptr[k]; i < T->pptr[k + 1]; ++i) cl[T->prods[i]].push_back((int)k);
    T->cptr.assign(1, 0);
    for (auto& c : cl) {
      T->cons.insert(T->cons.end(), c.begin(), c.end());
      T->cptr.push_back((int)T->cons.size());
    }
  }
  T->n_slots = n_slots;
  sizes[0] = (long long)tiles.size();
  sizes[1] = (long long)T->ent_tri.size();
  sizes[2] = T->band;
  sizes[3] = T->real;
  sizes[4] = T->lptr.back();
  sizes[5] = T->xptr.back();
  sizes[6] = T->n_slots;
  sizes[7] = T->n_halo;
  sizes[8] = T->pptr.back();
  *handle = T;
  return 0;
}

int hvb_tiling_fetch(void* handle, int* perm, int* tile_col0, int* tile_width, long long* tile_ptr, int* ent_tri,
                     int* ent_meta, int* tile_lptr, int* lcol, int* tile_xptr, int* xent, int* tile_pptr,
                     int* prods, int* tile_cptr, int* cons) {
  if (!handle) return 1;
  const Tiling* T = static_cast<const Tiling*>(handle);
  auto put = [](int* dst, const std::vector<int>& v) { std::memcpy(dst, v.data(), v.size() * sizeof(int)); };
  put(perm, T->perm);
  put(tile_col0, T->col0);
  put(tile_width, T->width);
  std::memcpy(tile_ptr, T->ptr.data(), T->ptr.size() * sizeof(long long));
  put(ent_tri, T->ent_tri);
  put(ent_meta, T->ent_meta);
  put(tile_lptr, T->lptr);
  put(lcol, T->lcol);
  put(tile_xptr, T->xptr);
  put(xent, T->xent);
  put(tile_pptr, T->pptr);
  put(prods, T->prods);
  put(tile_cptr, T->cptr);
  put(cons, T->cons);
  return 0;
}

int hvb_tiling_free(void* handle) {
  delete static_cast<Tiling*>(handle);
  return 0;
}

}  // extern "C"
