// Host planner of the B200 TSQR path: leaf tiles, the reduction tree and the
// launch schedule.  Product code (no oracle dependency).  The rules are those of
// row blocks of b rows (Eq. 1; remainder
// rule R6), tiles of <= s rows inside a block, binary reduction with the
// paper's pairing and promotion (Alg. TSQR:par; reading R5).
#pragma once
#include <cstdint>
#include <vector>

namespace tsqr {

struct PlanNode {
    int a, b;        // leftmost tiles of the left / right subtree; node id = b
    int stage;       // 0: tiles inside a row block, 1: row blocks of the rank
    int level;       // level inside its stage, from 1
    int step;        // global bottom-up step (all nodes of a step are independent)
};

struct Plan {
    int64_t m_local = 0, n = 0, b = 0, s = 0;
    int c = 32;                            // chunk rows of the tiles' flat chains
    std::vector<int64_t> tile_chunk0;      // first chunk of each tile (+ total)
    int nranks = 1, rank = 0;
    std::vector<int64_t> tile_row0, tile_rows;
    std::vector<int> blk_tile0;            // first tile of each row block (+ sentinel)
    std::vector<PlanNode> nodes;           // execution order
    std::vector<int> tile_parent;          // node id where leaf t is first merged, -1: none
    std::vector<int> node_a;               // by node id (b), [0] unused
    std::vector<int> node_parent;          // by node id, -1: the local root
    std::vector<int> node_step;            // by node id
    int nsteps = 0;
    int64_t max_rows = 0, min_rows = 0;
    int ntiles() const { return (int)tile_row0.size(); }
};

// Kernel tile capacity (rows) for a padded width, and the padded width of n.
int padded_width(int64_t n);
int64_t tile_capacity(int64_t n);
int64_t default_tile_rows(int64_t n);
int chunk_rows_for(int64_t n);

// Returns 0 on success, else a tsqr_status_t code.
int build_plan(int64_t m_local, int64_t n, int64_t block_rows, int64_t tile_rows,
               int nranks, int rank, Plan *out);

// Global slab of a rank.
int rank_slab(int64_t m, int64_t n, int64_t b, int nranks, int rank, int64_t *row0, int64_t *rows);

}  // namespace tsqr
