// Host-side job list of the single-layer pair-block kernel (k_blocks_slp) for
// a list of blocks: one pass in C++ instead of a chain of numpy passes (the
// coupling assembly of config 3 spent 0.3 s of host time there against 18 ms
// in the kernel).  Same output as the numpy restatement
// paper_2001_05523_b200.kernels.mirror_jobs, element for element
// (tests/test_host.py).

#include <cstdint>
#include <vector>

#include "h2b_internal.h"

using namespace h2b;

// For every block (t, s) of h_uids (n x 2) the index of block (s, t) in the
// same list, or -1; a diagonal block is its own partner.  Blocks are bucketed
// by row uid (counting sort), the partner found in row s's bucket.
extern "C" int h2b_block_partners(int64_t n, const int64_t* h_uids, int64_t* h_partner) {
    if (n < 0 || (n > 0 && (!h_uids || !h_partner))) return fail(H2B_ERR_INVALID, "h2b_block_partners: bad argument");
    if (n == 0) return ok();
    int64_t hi = 0;
    for (int64_t i = 0; i < 2 * n; ++i) {
        if (h_uids[i] < 0) return fail(H2B_ERR_INVALID, "h2b_block_partners: negative uid");
        if (h_uids[i] > hi) hi = h_uids[i];
    }
    std::vector<int64_t> ptr(hi + 2, 0), idx(n);
    for (int64_t i = 0; i < n; ++i) ++ptr[h_uids[2 * i] + 1];
    for (int64_t u = 0; u <= hi; ++u) ptr[u + 1] += ptr[u];
    {
        std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
        for (int64_t i = 0; i < n; ++i) idx[fill[h_uids[2 * i]]++] = i;
    }
    for (int64_t i = 0; i < n; ++i) {
        const int64_t t = h_uids[2 * i], s = h_uids[2 * i + 1];
        int64_t found = -1;
        // first match in list order (a block list holds every pair once)
        for (int64_t k = ptr[s]; k < ptr[s + 1]; ++k)
            if (h_uids[2 * idx[k] + 1] == t) {
                found = idx[k];
                break;
            }
        h_partner[i] = found;
    }
    return ok();
}

// Jobs (row_off, n_rows, col_off, n_cols, out_off, ld, mirror_off, mirror_ld)
// of n blocks (t, s) = h_uids[i]: rows row_off[t] .. + row_cnt[t] of the row
// index list, columns col_off[s] .. + col_cnt[s] of the column index list,
// written at blk_off[i] with leading dimension blk_ld[i].  mirrored != 0
// (symmetric single layer: block (s, t) = block (t, s)^T) keeps one job per
// block pair -- the block with t <= s, or a block without partner -- which
// also writes its transpose at the partner's place; otherwise one job per
// block with mirror_off = -1, mirror_ld = 0.  h_jobs holds 8 n words; the
// number of jobs kept is returned in h_n_jobs.
extern "C" int h2b_block_jobs(int64_t n, const int64_t* h_uids, const int64_t* h_row_off, const int64_t* h_row_cnt,
                              const int64_t* h_col_off, const int64_t* h_col_cnt, const int64_t* h_blk_off,
                              const int64_t* h_blk_ld, int mirrored, const int64_t* h_partner, int64_t* h_jobs,
                              int64_t* h_n_jobs) {
    if (n < 0 || !h_n_jobs) return fail(H2B_ERR_INVALID, "h2b_block_jobs: bad argument");
    *h_n_jobs = 0;
    if (n == 0) return ok();
    if (!h_uids || !h_row_off || !h_row_cnt || !h_col_off || !h_col_cnt || !h_blk_off || !h_blk_ld || !h_jobs ||
        (mirrored && !h_partner))
        return fail(H2B_ERR_INVALID, "h2b_block_jobs: null pointer");
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t t = h_uids[2 * i], s = h_uids[2 * i + 1];
        const int64_t p = mirrored ? h_partner[i] : -1;
        if (p >= n) return fail(H2B_ERR_INVALID, "h2b_block_jobs: partner index out of range");
        if (mirrored && p >= 0 && t > s) continue;  // written by its partner's job
        int64_t* j = h_jobs + 8 * m++;
        j[0] = h_row_off[t];
        j[1] = h_row_cnt[t];
        j[2] = h_col_off[s];
        j[3] = h_col_cnt[s];
        j[4] = h_blk_off[i];
        j[5] = h_blk_ld[i];
        j[6] = p >= 0 ? h_blk_off[p] : -1;
        j[7] = p >= 0 ? h_blk_ld[p] : 0;
    }
    *h_n_jobs = m;
    return ok();
}
