// host_neighbors.cpp -- host-side ordered nearest-predecessor search (C ABI, OpenMP).
//
// The neighbor table is an INPUT of the GPU path and stays on the host (BASELINE.json
// north_star); it must equal the reference's table entry for entry.  The reference
// defines it by an exhaustive scan (/root/reference/pkg/src/vecchiagp/engine/
// _kernels.pyx:609-651, preprocess.py:121-132): row i = i followed by the m
// predecessors j < i with the smallest (d2, j) in lexicographic order, where
// d2 = sum over axes of (x_i - x_j)^2 accumulated left to right in double precision
// WITHOUT fused multiply-add (pkg/setup.py:18-25).  That scan is O(n^2) -- hours at
// n >= 2^22 -- so this file provides the same table from a multi-resolution uniform
// grid: candidates are enumerated ring by ring around the query cell and ranked with
// the identical d2 expression and tie rule, and the search stops only when no
// unvisited cell can hold a point that beats or ties the current m-th best.
// Build with -ffp-contract=off (see build.py) so d2 is bit-identical.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct Cand {
    double d2;
    int64_t j;
};

inline bool before(double d2a, int64_t ja, double d2b, int64_t jb) { return d2a < d2b || (d2a == d2b && ja < jb); }

// bounded sorted list of the m best (d2, j) keys
struct Best {
    Cand *v;
    int m, cnt;
    inline double worst() const { return v[m - 1].d2; }
    inline int64_t worst_j() const { return v[m - 1].j; }
    inline void offer(double d2, int64_t j)
    {
        if (cnt == m && !before(d2, j, v[m - 1].d2, v[m - 1].j))
            return;
        int pos = cnt < m ? cnt++ : m - 1;
        while (pos > 0 && before(d2, j, v[pos - 1].d2, v[pos - 1].j)) {
            v[pos] = v[pos - 1];
            --pos;
        }
        v[pos].d2 = d2;
        v[pos].j = j;
    }
};

inline double sqdist(const double *a, const double *b, int d)
{
    double s = 0.0;
    for (int l = 0; l < d; ++l) {
        const double diff = a[l] - b[l];
        s += diff * diff;
    }
    return s;
}

// One grid level: the first `count` points binned on the first g axes.
struct Level {
    int64_t count = 0;
    int g = 0;
    int dims[3] = {1, 1, 1};
    double h = 1.0, inv_h = 1.0;
    std::vector<int64_t> start; // cell -> first slot
    std::vector<int32_t> items; // point indices, ascending inside a cell
};

struct Grid {
    int g;
    double lo[3], ext[3];
    std::vector<Level> levels;
    std::vector<int64_t> level_count;
};

inline void cell_of(const Level &L, const Grid &G, const double *x, int *c)
{
    for (int a = 0; a < 3; ++a) {
        if (a < L.g) {
            int v = (int)std::floor((x[a] - G.lo[a]) * L.inv_h);
            c[a] = v < 0 ? 0 : (v >= L.dims[a] ? L.dims[a] - 1 : v);
        } else {
            c[a] = 0;
        }
    }
}

void build_level(Level &L, const Grid &G, const double *locs, int d, int64_t count, double per_cell)
{
    L.count = count;
    L.g = G.g;
    double vol = 1.0;
    int live = 0;
    for (int a = 0; a < G.g; ++a)
        if (G.ext[a] > 0.0) {
            vol *= G.ext[a];
            ++live;
        }
    double h = live ? std::pow(vol * per_cell / (double)count, 1.0 / live) : 1.0;
    if (!(h > 0.0) || !std::isfinite(h))
        h = 1.0;
    // cap the number of cells
    for (;;) {
        double cells = 1.0;
        for (int a = 0; a < G.g; ++a)
            cells *= std::floor(G.ext[a] / h) + 1.0;
        if (cells <= 4.0 * (double)count + 64.0)
            break;
        h *= 1.5;
    }
    L.h = h;
    L.inv_h = 1.0 / h;
    int64_t ncell = 1;
    for (int a = 0; a < 3; ++a) {
        L.dims[a] = a < G.g ? (int)std::floor(G.ext[a] / h) + 1 : 1;
        ncell *= L.dims[a];
    }
    L.start.assign((size_t)ncell + 1, 0);
    std::vector<int64_t> cid((size_t)count);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        int c[3];
        cell_of(L, G, locs + i * d, c);
        cid[i] = ((int64_t)c[2] * L.dims[1] + c[1]) * L.dims[0] + c[0];
    }
    for (int64_t i = 0; i < count; ++i)
        L.start[cid[i] + 1]++;
    for (int64_t c = 0; c < ncell; ++c)
        L.start[c + 1] += L.start[c];
    L.items.resize((size_t)count);
    std::vector<int64_t> fill(L.start.begin(), L.start.end() - 1);
    for (int64_t i = 0; i < count; ++i) // ascending i keeps each cell sorted by index
        L.items[fill[cid[i]]++] = (int32_t)i;
}

void exhaustive_row(const double *locs, int d, int64_t i, Best &B)
{
    const double *xi = locs + i * d;
    for (int64_t j = 0; j < i; ++j)
        B.offer(sqdist(xi, locs + j * d, d), j);
}

void grid_row(const Grid &G, const Level &L, const double *locs, int d, int64_t i, Best &B)
{
    const double *xi = locs + i * d;
    int cq[3];
    cell_of(L, G, xi, cq);
    int maxr = 0;
    for (int a = 0; a < L.g; ++a)
        maxr = std::max(maxr, std::max(cq[a], L.dims[a] - 1 - cq[a]));
    for (int r = 0; r <= maxr; ++r) {
        if (r >= 1 && B.cnt == B.m) {
            // every unvisited cell is at least r cells away along some axis: its points are
            // farther than (r-1)*h + (distance to the own cell face) >= (r-1)*h ... use the
            // conservative bound with a relative safety margin for the floor() rounding.
            const double lb = (double)(r - 1) * L.h * 0.999999;
            if (r >= 2 && B.worst() < lb * lb)
                break;
        }
        const int z0 = L.g > 2 ? std::max(cq[2] - r, 0) : 0, z1 = L.g > 2 ? std::min(cq[2] + r, L.dims[2] - 1) : 0;
        const int y0 = L.g > 1 ? std::max(cq[1] - r, 0) : 0, y1 = L.g > 1 ? std::min(cq[1] + r, L.dims[1] - 1) : 0;
        const int x0 = std::max(cq[0] - r, 0), x1 = std::min(cq[0] + r, L.dims[0] - 1);
        for (int z = z0; z <= z1; ++z) {
            const bool zface = L.g > 2 && (z == cq[2] - r || z == cq[2] + r);
            for (int y = y0; y <= y1; ++y) {
                const bool yface = L.g > 1 && (y == cq[1] - r || y == cq[1] + r);
                const int64_t rowbase = ((int64_t)z * L.dims[1] + y) * L.dims[0];
                if (zface || yface) {
                    // whole x-run belongs to the shell
                    const int64_t s = L.start[rowbase + x0], e = L.start[rowbase + x1 + 1];
                    for (int64_t t = s; t < e; ++t) {
                        const int64_t j = L.items[t];
                        if (j >= i)
                            continue;
                        B.offer(sqdist(xi, locs + j * d, d), j);
                    }
                } else {
                    // only the two x faces
                    for (int side = 0; side < 2; ++side) {
                        const int x = side ? cq[0] + r : cq[0] - r;
                        if (x < 0 || x >= L.dims[0] || (side && r == 0))
                            continue;
                        const int64_t s = L.start[rowbase + x], e = L.start[rowbase + x + 1];
                        for (int64_t t = s; t < e; ++t) {
                            const int64_t j = L.items[t];
                            if (j >= i)
                                continue;
                            B.offer(sqdist(xi, locs + j * d, d), j);
                        }
                    }
                }
            }
        }
    }
}

// ring search around an arbitrary query point (all points of the level are candidates).  The squared
// distance is evaluated as (train - query), matching the reference's `work_train - point`.
void grid_query(const Grid &G, const Level &L, const double *locs, int d, const double *xq, Best &B)
{
    int cq[3];
    cell_of(L, G, xq, cq);
    // distance by which the query lies outside the box along each gridded axis (0 inside)
    double out2 = 0.0;
    for (int a = 0; a < L.g; ++a) {
        const double below = G.lo[a] - xq[a], above = xq[a] - (G.lo[a] + G.ext[a]);
        const double o = below > 0.0 ? below : (above > 0.0 ? above : 0.0);
        out2 = o > out2 ? o : out2;
    }
    (void)out2;
    int maxr = 0;
    for (int a = 0; a < L.g; ++a)
        maxr = std::max(maxr, std::max(cq[a], L.dims[a] - 1 - cq[a]));
    for (int r = 0; r <= maxr; ++r) {
        if (r >= 2 && B.cnt == B.m) {
            const double lb = (double)(r - 1) * L.h * 0.999999;
            if (B.worst() < lb * lb)
                break;
        }
        const int z0 = L.g > 2 ? std::max(cq[2] - r, 0) : 0, z1 = L.g > 2 ? std::min(cq[2] + r, L.dims[2] - 1) : 0;
        const int y0 = L.g > 1 ? std::max(cq[1] - r, 0) : 0, y1 = L.g > 1 ? std::min(cq[1] + r, L.dims[1] - 1) : 0;
        const int x0 = std::max(cq[0] - r, 0), x1 = std::min(cq[0] + r, L.dims[0] - 1);
        for (int z = z0; z <= z1; ++z) {
            const bool zface = L.g > 2 && (z == cq[2] - r || z == cq[2] + r);
            for (int y = y0; y <= y1; ++y) {
                const bool yface = L.g > 1 && (y == cq[1] - r || y == cq[1] + r);
                const int64_t rowbase = ((int64_t)z * L.dims[1] + y) * L.dims[0];
                if (zface || yface) {
                    const int64_t s = L.start[rowbase + x0], e = L.start[rowbase + x1 + 1];
                    for (int64_t t = s; t < e; ++t) {
                        const int64_t j = L.items[t];
                        B.offer(sqdist(locs + j * d, xq, d), j);
                    }
                } else {
                    for (int side = 0; side < 2; ++side) {
                        const int x = side ? cq[0] + r : cq[0] - r;
                        if (x < 0 || x >= L.dims[0] || (side && r == 0))
                            continue;
                        const int64_t s = L.start[rowbase + x], e = L.start[rowbase + x + 1];
                        for (int64_t t = s; t < e; ++t) {
                            const int64_t j = L.items[t];
                            B.offer(sqdist(locs + j * d, xq, d), j);
                        }
                    }
                }
            }
        }
    }
}

} // namespace

extern "C" {

int vbh_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// Exhaustive scan (the normative algorithm).  out is (n, m+1) int64.
int vbh_neighbors_exhaustive(const double *locs, int64_t n, int d, int m, int workers, int64_t *out)
{
    if (!locs || !out || n < 1 || d < 1 || m < 1)
        return -1;
    if (workers < 1)
        workers = 1;
#pragma omp parallel num_threads(workers)
    {
        std::vector<Cand> buf((size_t)m);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            Best B{buf.data(), m, 0};
            exhaustive_row(locs, d, i, B);
            int64_t *row = out + i * (m + 1);
            row[0] = i;
            for (int t = 0; t < m; ++t)
                row[1 + t] = t < B.cnt ? B.v[t].j : -1;
        }
    }
    return 0;
}

// Grid-accelerated search of rows [row0, row0 + rows) only; out is (rows, m+1).  Identical
// output to the corresponding rows of vbh_neighbors_exhaustive.  Each rank of a multi-GPU
// run builds just its own shard of the table with this entry point.
int vbh_neighbors_grid_rows(const double *locs, int64_t n, int d, int m, int workers, int64_t row0, int64_t rows,
                            int64_t *out)
{
    if (!locs || !out || n < 1 || d < 1 || m < 1 || row0 < 0 || rows < 0 || row0 + rows > n)
        return -1;
    if (n > (int64_t)0x7fffffff)
        return -2;
    if (workers < 1)
        workers = 1;
    for (int64_t t = 0; t < n * d; ++t)
        if (!std::isfinite(locs[t]))
            return -3;
    Grid G;
    G.g = d < 3 ? d : 3;
    for (int a = 0; a < G.g; ++a) {
        double lo = locs[a], hi = locs[a];
        for (int64_t i = 1; i < n; ++i) {
            const double v = locs[i * d + a];
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
        G.lo[a] = lo;
        G.ext[a] = hi - lo;
    }
    // levels cover prefixes of length base * 2^l; rows below `base` are scanned exhaustively
    const int64_t base = std::max<int64_t>(1024, 16 * (int64_t)m);
    const double per_cell = std::max(3.0, 0.35 * m);
    for (int64_t c = 2 * base; ; c *= 2) {
        const int64_t cnt = std::min(c, n);
        if (cnt <= base)
            break;
        G.level_count.push_back(cnt);
        if (cnt == n)
            break;
    }
    G.levels.resize(G.level_count.size());
    for (size_t l = 0; l < G.levels.size(); ++l)
        build_level(G.levels[l], G, locs, d, G.level_count[l], per_cell);
#pragma omp parallel num_threads(workers)
    {
        std::vector<Cand> buf((size_t)m);
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = row0; i < row0 + rows; ++i) {
            Best B{buf.data(), m, 0};
            if (i <= base || G.levels.empty()) {
                exhaustive_row(locs, d, i, B);
            } else {
                size_t l = 0;
                while (G.level_count[l] < i)
                    ++l;
                grid_row(G, G.levels[l], locs, d, i, B);
            }
            int64_t *row = out + (i - row0) * (m + 1);
            row[0] = i;
            for (int t = 0; t < m; ++t)
                row[1 + t] = t < B.cnt ? B.v[t].j : -1;
        }
    }
    return 0;
}

// m nearest TRAINING points (no ordering constraint) of each query point, ranked by (d2, index)
// -- the selection rule of the reference's kriging (predict.py:27-32, np.lexsort((index, d2))).
// out is (nq, m) int64.  Same grid machinery: one level holding all n points.
int vbh_neighbors_query(const double *locs, int64_t n, int d, const double *queries, int64_t nq, int m, int workers,
                        int64_t *out)
{
    if (!locs || !queries || !out || n < 1 || d < 1 || m < 1 || m > n || nq < 0)
        return -1;
    if (n > (int64_t)0x7fffffff)
        return -2;
    if (workers < 1)
        workers = 1;
    Grid G;
    G.g = d < 3 ? d : 3;
    for (int a = 0; a < G.g; ++a) {
        double lo = locs[a], hi = locs[a];
        for (int64_t i = 1; i < n; ++i) {
            const double v = locs[i * d + a];
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
        G.lo[a] = lo;
        G.ext[a] = hi - lo;
    }
    const bool use_grid = n > 2048;
    Level L;
    if (use_grid)
        build_level(L, G, locs, d, n, std::max(3.0, 0.35 * m));
#pragma omp parallel num_threads(workers)
    {
        std::vector<Cand> buf((size_t)m);
#pragma omp for schedule(dynamic, 64)
        for (int64_t t = 0; t < nq; ++t) {
            Best B{buf.data(), m, 0};
            const double *xq = queries + t * d;
            if (!use_grid) {
                for (int64_t j = 0; j < n; ++j)
                    B.offer(sqdist(locs + j * d, xq, d), j);
            } else {
                // a query outside the bounding box is clamped into the border cell; its true distance to
                // any cell is then larger than the in-grid bound used by the stopping rule (conservative)
                grid_query(G, L, locs, d, xq, B);
            }
            for (int k = 0; k < m; ++k)
                out[t * m + k] = k < B.cnt ? B.v[k].j : -1;
        }
    }
    return 0;
}

// Max-min distance ordering (BASELINE.json config 1 names it, the reference has
// only identity / random orderings).  Definition: perm[0] = the point nearest the coordinate-wise
// mean (smallest index on ties); perm[k] = the not-yet-chosen point whose minimum distance to
// {perm[0..k-1]} is largest (smallest index on ties).  Exact greedy selection in ~O(n log n): every
// point keeps its current min squared distance d[j]; a lazy max-heap yields the next point i*, and
// only points within sqrt(d[i*]) of i* can have their d[j] lowered (all d[j] <= d[i*]), which a
// uniform grid enumerates.  out receives the permutation (new position -> original index).
int vbh_order_maxmin(const double *locs, int64_t n, int d, int64_t *out)
{
    if (!locs || !out || n < 1 || d < 1)
        return -1;
    if (n > (int64_t)0x7fffffff)
        return -2;
    for (int64_t t = 0; t < n * d; ++t)
        if (!std::isfinite(locs[t]))
            return -3;
    // first point: nearest to the centroid
    std::vector<double> mean((size_t)d, 0.0);
    for (int64_t i = 0; i < n; ++i)
        for (int l = 0; l < d; ++l)
            mean[l] += locs[i * d + l];
    for (int l = 0; l < d; ++l)
        mean[l] /= (double)n;
    int64_t first = 0;
    double best = sqdist(locs, mean.data(), d);
    for (int64_t i = 1; i < n; ++i) {
        const double v = sqdist(locs + i * d, mean.data(), d);
        if (v < best) {
            best = v;
            first = i;
        }
    }
    Grid G;
    G.g = d < 3 ? d : 3;
    for (int a = 0; a < G.g; ++a) {
        double lo = locs[a], hi = locs[a];
        for (int64_t i = 1; i < n; ++i) {
            const double v = locs[i * d + a];
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
        G.lo[a] = lo;
        G.ext[a] = hi - lo;
    }
    Level L;
    build_level(L, G, locs, d, n, 3.0);
    std::vector<int64_t> fill(L.start.begin() + 1, L.start.end()); // live end of every cell (swap-remove)
    std::vector<int32_t> slot((size_t)n);                          // position of a point inside items
    for (int64_t c = 0; c + 1 < (int64_t)L.start.size(); ++c)
        for (int64_t t = L.start[c]; t < L.start[c + 1]; ++t)
            slot[L.items[t]] = (int32_t)t;
    auto remove_point = [&](int64_t i) {
        int c[3];
        cell_of(L, G, locs + i * d, c);
        const int64_t cell = ((int64_t)c[2] * L.dims[1] + c[1]) * L.dims[0] + c[0];
        const int64_t pos = slot[i], last = --fill[cell];
        const int32_t moved = L.items[last];
        L.items[pos] = moved;
        slot[moved] = (int32_t)pos;
        L.items[last] = (int32_t)i;
    };
    std::vector<double> dmin((size_t)n);
    typedef std::pair<double, int64_t> Key; // (d, -index): max-heap pops the largest d, smallest index on ties
    std::vector<Key> heap;
    heap.reserve((size_t)n * 2);
    for (int64_t i = 0; i < n; ++i) {
        dmin[i] = sqdist(locs + i * d, locs + first * d, d);
        if (i != first)
            heap.emplace_back(dmin[i], -i);
    }
    std::make_heap(heap.begin(), heap.end());
    std::vector<char> chosen((size_t)n, 0);
    chosen[first] = 1;
    remove_point(first);
    out[0] = first;
    for (int64_t k = 1; k < n; ++k) {
        int64_t pick = -1;
        double r2 = 0.0;
        while (!heap.empty()) {
            std::pop_heap(heap.begin(), heap.end());
            const Key top = heap.back();
            heap.pop_back();
            const int64_t i = -top.second;
            if (!chosen[i] && top.first == dmin[i]) {
                pick = i;
                r2 = top.first;
                break;
            }
        }
        if (pick < 0)
            return -4;
        out[k] = pick;
        chosen[pick] = 1;
        remove_point(pick);
        // lower d[j] of the live points within sqrt(r2) of the pick
        const double *xp = locs + pick * d;
        const double r = std::sqrt(r2) * 1.000001 + 1e-300;
        int c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};
        for (int a = 0; a < L.g; ++a) {
            int lo = (int)std::floor((xp[a] - r - G.lo[a]) * L.inv_h), hi = (int)std::floor((xp[a] + r - G.lo[a]) * L.inv_h);
            c0[a] = lo < 0 ? 0 : (lo >= L.dims[a] ? L.dims[a] - 1 : lo);
            c1[a] = hi < 0 ? 0 : (hi >= L.dims[a] ? L.dims[a] - 1 : hi);
        }
        for (int z = c0[2]; z <= c1[2]; ++z)
            for (int y = c0[1]; y <= c1[1]; ++y) {
                const int64_t rowbase = ((int64_t)z * L.dims[1] + y) * L.dims[0];
                for (int x = c0[0]; x <= c1[0]; ++x) {
                    const int64_t cell = rowbase + x;
                    for (int64_t t = L.start[cell]; t < fill[cell]; ++t) {
                        const int64_t j = L.items[t];
                        const double v = sqdist(locs + j * d, xp, d);
                        if (v < dmin[j]) {
                            dmin[j] = v;
                            heap.emplace_back(v, -j);
                            std::push_heap(heap.begin(), heap.end());
                        }
                    }
                }
            }
    }
    return 0;
}

// Grid-accelerated search of the whole table; identical output to vbh_neighbors_exhaustive.
int vbh_neighbors_grid(const double *locs, int64_t n, int d, int m, int workers, int64_t *out)
{
    return vbh_neighbors_grid_rows(locs, n, d, m, workers, 0, n, out);
}

// Dependency levels of the ordered-neighbor DAG (row i conditions on earlier rows only): level(i) =
// 1 + max level of its neighbors, 0 for a row without neighbors.  Observations of one level are mutually
// independent given the lower levels -- the schedule of the device conditional simulator.
// order (n): observation indices sorted by (level, index); level_ptr (n + 1 entries allocated by the
// caller, nlevels + 1 used): order[level_ptr[l] .. level_ptr[l+1]) is level l.  Returns nlevels, -1 on a
// malformed table (a neighbor index >= its row).
int64_t vbh_dependency_levels(const int64_t *nn, int64_t n, int mp1, int64_t *order, int64_t *level_ptr)
{
    std::vector<int32_t> level((size_t)n);
    int64_t nlev = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t lv = 0;
        const int64_t *row = nn + i * mp1;
        for (int c = 1; c < mp1; ++c) {
            const int64_t j = row[c];
            if (j < 0)
                break;
            if (j >= i)
                return -1;
            lv = std::max(lv, level[(size_t)j] + 1);
        }
        level[(size_t)i] = lv;
        nlev = std::max<int64_t>(nlev, lv + 1);
    }
    for (int64_t l = 0; l <= nlev; ++l)
        level_ptr[l] = 0;
    for (int64_t i = 0; i < n; ++i)
        ++level_ptr[level[(size_t)i] + 1];
    for (int64_t l = 0; l < nlev; ++l)
        level_ptr[l + 1] += level_ptr[l];
    std::vector<int64_t> cursor(level_ptr, level_ptr + nlev);
    for (int64_t i = 0; i < n; ++i)
        order[cursor[(size_t)level[(size_t)i]]++] = i;
    return nlev;
}

// Narrow a block of neighbor indices (int64, -1 = padding) to int32 for the host-to-device transfer: the table is
// 8(m+1) bytes per observation and the end-to-end path is bound by the PCIe copy of it; indices of any dataset with
// n < 2^31 points fit 32 bits, the device widens them back (vb200_widen_indices).  All host threads; returns 0, or
// 1 if some value does not fit (the caller then ships the int64 rows as they are).
int vbh_narrow_indices(const int64_t *src, int32_t *dst, int64_t count, int workers)
{
    if (!src || !dst || count < 0)
        return -1;
    int bad = 0;
#ifdef _OPENMP
    if (workers < 1)
        workers = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(workers) reduction(| : bad)
#endif
    for (int64_t i = 0; i < count; ++i) {
        const int64_t v = src[i];
        dst[i] = (int32_t)v;
        bad |= (v != (int64_t)(int32_t)v);
    }
    return bad;
}

} // extern "C"
