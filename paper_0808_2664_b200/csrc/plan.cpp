// Host planner (see plan.h).  The binary reduction over an ordered list is
// written in stride form: at level l the survivor at list index i (i divisible
// by 2^l) absorbs index i + 2^(l-1) when that index exists -- the same tree as
// pairing (2q, 2q+1) on the compacted list with the odd tail promoted.
#include "plan.h"
#include "../../include/tsqr.h"

#include <algorithm>

namespace tsqr {

int padded_width(int64_t n) { return n <= 16 ? 16 : (n <= 32 ? 32 : 64); }

// A tile is factored as a flat chain of register-resident chunks (chunk.cuh),
// so its height is bounded only by the 32-bit row count of the device plan.
// Default tile: 32 chunks of the chain.
// Wide n (> 64): the leaf is one blocked QR of the whole tile by one CTA, at
// most 2304 logical rows (tsqr_wide.cu), default 2048.
int64_t tile_capacity(int64_t n) { return n > 64 ? 2304 : (int64_t)1 << 30; }
int64_t default_tile_rows(int64_t n) { return n > 64 ? 2048 : 32 * (int64_t)chunk_rows_for(n); }
// chunk.cuh: the chunk is register-resident (KM x NCB DMMA fragments per lane),
// as tall as the register file and the staging buffers allow at 8 warps/SM:
// KM = 8 (64 rows) for n <= 32, 6 (48) for n <= 48, 5 (40) for n <= 64 (for
// 56 < n <= 64 with a single R buffer, tsqr_chain.cu)
#ifndef TSQR_C32
#define TSQR_C32 64
#endif
int chunk_rows_for(int64_t n) {
    return n <= 16 ? 64 : (n <= 32 ? TSQR_C32 : (n <= 48 ? 48 : (n <= 64 ? 40 : 0)));   // 0: one chunk per tile
}

static int64_t block_count(int64_t m, int64_t n, int64_t b, int64_t *last_rows) {
    // Reading R6: blocks of b rows; a remainder >= n is its own block, a
    // shorter one is merged into the last block.
    int64_t full = m / b, rem = m % b;
    if (full == 0) { *last_rows = m; return 1; }
    if (rem == 0) { *last_rows = b; return full; }
    if (rem >= n) { *last_rows = rem; return full + 1; }
    *last_rows = b + rem;
    return full;
}

int rank_slab(int64_t m, int64_t n, int64_t b, int nranks, int rank, int64_t *row0, int64_t *rows) {
    if (n < 1 || m < n || b < 1) return TSQR_ERR_SHAPE;
    if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks) return TSQR_ERR_INVALID;
    int64_t last = 0;
    int64_t nb = block_count(m, n, b, &last);
    if (nb < nranks) return TSQR_ERR_SHAPE;
    int64_t q = nb / nranks, extra = nb % nranks;
    int64_t first_blk = rank * q + std::min<int64_t>(rank, extra);
    int64_t my_blocks = q + (rank < extra ? 1 : 0);
    *row0 = first_blk * b;
    bool has_last = (first_blk + my_blocks == nb);
    *rows = has_last ? (my_blocks - 1) * b + last : my_blocks * b;
    return TSQR_OK;
}

// Binary reduction over `items` (tile ids, leftmost of each subtree).
static void reduce(const std::vector<int> &items, int stage, std::vector<PlanNode> &out) {
    const int len = (int)items.size();
    for (int level = 1, half = 1; half < len; ++level, half *= 2)
        for (int i = 0; i + half < len; i += 2 * half)
            out.push_back(PlanNode{items[i], items[i + half], stage, level, 0});
}

int build_plan(int64_t m_local, int64_t n, int64_t block_rows, int64_t tile_rows,
               int nranks, int rank, Plan *p) {
    if (n < 1 || m_local < n) return TSQR_ERR_SHAPE;
    if (n > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    if (block_rows < 1 || tile_rows < 0) return TSQR_ERR_INVALID;
    if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks) return TSQR_ERR_UNSUPPORTED;
    const int64_t cap = tile_capacity(n);
    const int64_t s = tile_rows == 0 ? std::min(default_tile_rows(n), block_rows) : tile_rows;
    if (s > cap) return TSQR_ERR_UNSUPPORTED;

    *p = Plan();
    p->m_local = m_local; p->n = n; p->b = block_rows; p->s = s;
    p->nranks = nranks; p->rank = rank;

    int64_t last = 0;
    const int64_t nblk = block_count(m_local, n, block_rows, &last);
    if (nblk > (int64_t)1 << 30) return TSQR_ERR_UNSUPPORTED;
    int64_t row = 0;
    for (int64_t k = 0; k < nblk; ++k) {
        const int64_t h = (k == nblk - 1) ? last : block_rows;
        // tiles of near-equal height, never shorter than n
        const int64_t t = std::max<int64_t>(1, std::min<int64_t>((h + s - 1) / s, h / n));
        p->blk_tile0.push_back((int)p->tile_row0.size());
        // even heights when every tile keeps >= n rows (row pairs split near-equally, the
        // last tile takes the rest): with an even block start every tile then starts on an
        // even row, as the leaf kernel's TMA staging needs
        const int64_t pb = (h / 2) / t, pe = (h / 2) % t;
        const int64_t last_even = h - 2 * (pb * (t - 1) + std::min<int64_t>(pe, t - 1));
        const bool even = t > 1 && 2 * pb >= n && last_even >= n;
        for (int64_t i = 0; i < t; ++i) {
            const int64_t rows = even ? (i < t - 1 ? 2 * (pb + (i < pe ? 1 : 0)) : last_even)
                                      : h / t + (i < h % t ? 1 : 0);
            if (rows < n) return TSQR_ERR_SHAPE;
            if (rows > cap) return TSQR_ERR_UNSUPPORTED;
            p->tile_row0.push_back(row);
            p->tile_rows.push_back(rows);
            row += rows;
        }
    }
    p->blk_tile0.push_back((int)p->tile_row0.size());
    if ((int64_t)p->tile_row0.size() > ((int64_t)1 << 31) - 1) return TSQR_ERR_UNSUPPORTED;
    const int L = p->ntiles();
    p->c = chunk_rows_for(n);
    p->tile_chunk0.assign(L + 1, 0);
    for (int t = 0; t < L; ++t)
        p->tile_chunk0[t + 1] = p->tile_chunk0[t] + (p->c > 0 ? (p->tile_rows[t] + p->c - 1) / p->c : 1);
    p->max_rows = *std::max_element(p->tile_rows.begin(), p->tile_rows.end());
    p->min_rows = *std::min_element(p->tile_rows.begin(), p->tile_rows.end());

    // stage 0: a tree inside every block; stage 1: a tree over the blocks.
    for (int64_t k = 0; k < nblk; ++k) {
        std::vector<int> items;
        for (int t = p->blk_tile0[k]; t < p->blk_tile0[k + 1]; ++t) items.push_back(t);
        reduce(items, 0, p->nodes);
    }
    {
        std::vector<int> items(p->blk_tile0.begin(), p->blk_tile0.end() - 1);
        reduce(items, 1, p->nodes);
    }
    // Steps: every stage-0 level l is step l, stage-1 level l is step D0 + l.
    int d0 = 0;
    for (auto &nd : p->nodes) if (nd.stage == 0) d0 = std::max(d0, nd.level);
    for (auto &nd : p->nodes) {
        nd.step = nd.stage == 0 ? nd.level : d0 + nd.level;
        p->nsteps = std::max(p->nsteps, nd.step);
    }
    // Parent links.  A subtree is named by its leftmost tile; the nodes that
    // tile takes part in, in execution order, are: every node where it is the
    // left child, then (possibly) the node where it is the right child.
    p->tile_parent.assign(L, -1);
    p->node_a.assign(L, -1);
    p->node_parent.assign(L, -1);
    p->node_step.assign(L, 0);
    std::vector<int> last_node_of(L, -1);     // the last node seen for each leftmost tile
    for (const auto &nd : p->nodes) {
        p->node_a[nd.b] = nd.a;
        p->node_step[nd.b] = nd.step;
        for (int child : {nd.a, nd.b}) {
            if (last_node_of[child] < 0) p->tile_parent[child] = nd.b;
            else p->node_parent[last_node_of[child]] = nd.b;
        }
        last_node_of[nd.a] = nd.b;
    }
    return TSQR_OK;
}

}  // namespace tsqr
