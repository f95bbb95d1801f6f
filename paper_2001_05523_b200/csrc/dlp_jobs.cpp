// Host-side DLP job builder (the reference's column-panel sets of
// kernels.panel_pair_matrix / dlp_block, kernels.py:448-468, tiled for
// k_blocks_dlp).  Same output as the Python restatement
// paper_2001_05523_b200.kernels._build_dlp_jobs_py, element for element
// (tests/test_host.py), ~100x faster: the DLP assembly of config 2 spends its
// host time here.

#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "h2b_internal.h"

namespace {
constexpr int64_t kTile = 64;       // rows / columns of one job (kernel tile)
constexpr int64_t kMaxPanels = 128; // panels of one job (kernel shared memory)
}  // namespace

struct h2b_dlp_build {
    std::vector<int64_t> jobs;      // 8 words per job
    std::vector<int32_t> row_idx, pan_idx, inc_ptr, inc;
    std::vector<int64_t> inc_base;
};

using namespace h2b;

namespace {
// Jobs of blocks [b0, b1) with offsets local to this range (0-based row_idx,
// pan_idx, inc and incidence-pointer lists); merged in block order below.
int build_range(int64_t n_verts, const int64_t* vptr, const int64_t* vidx, const int64_t* tris, int64_t b0,
                int64_t b1, const int64_t* row_ptr, const int64_t* rows, const int64_t* col_ptr,
                const int64_t* cols, const int64_t* out_off, const int64_t* ld, h2b_dlp_build* b,
                std::string& err) {
    std::vector<int32_t> vpos((size_t)std::max<int64_t>(n_verts, 0), -1);
    std::vector<int64_t> pans;
    struct Trip {
        int32_t c, l, p;
    };
    std::vector<Trip> trip;
    int64_t nrow = 0, npan = 0, ninc = 0, nptr = 0;
    for (int64_t bk = b0; bk < b1; ++bk) {
        const int64_t* R = rows + row_ptr[bk];
        const int64_t nr = row_ptr[bk + 1] - row_ptr[bk];
        const int64_t* Cc = cols + col_ptr[bk];
        const int64_t ncol = col_ptr[bk + 1] - col_ptr[bk];
        int64_t c0 = 0;
        while (c0 < ncol) {
            int64_t c1 = std::min(ncol, c0 + kTile);
            while (true) {  // the column tile, halved until its panel set fits
                pans.clear();
                for (int64_t c = c0; c < c1; ++c) {
                    const int64_t v = Cc[c];
                    if (v < 0 || v >= n_verts) {
                        err = "h2b_dlp_jobs_build: column vertex out of range";
                        return H2B_ERR_INVALID;
                    }
                    pans.insert(pans.end(), vidx + vptr[v], vidx + vptr[v + 1]);
                }
                std::sort(pans.begin(), pans.end());
                pans.erase(std::unique(pans.begin(), pans.end()), pans.end());
                if ((int64_t)pans.size() <= kMaxPanels || c1 - c0 == 1) break;
                c1 = c0 + std::max<int64_t>(1, (c1 - c0) / 2);
            }
            if ((int64_t)pans.size() > kMaxPanels) {
                err = "vertex valence too large for the DLP panel tile";
                return H2B_ERR_INVALID;
            }
            const int64_t nsel = c1 - c0;
            for (int64_t c = c0; c < c1; ++c) vpos[Cc[c]] = (int32_t)(c - c0);
            trip.clear();
            const int64_t np = (int64_t)pans.size();
            for (int l = 0; l < 3; ++l)
                for (int64_t p = 0; p < np; ++p) {
                    const int32_t c = vpos[tris[3 * pans[p] + l]];
                    if (c >= 0) trip.push_back({c, l, (int32_t)p});
                }
            for (int64_t c = c0; c < c1; ++c) vpos[Cc[c]] = -1;
            std::sort(trip.begin(), trip.end(), [](const Trip& x, const Trip& y) {
                return x.c != y.c ? x.c < y.c : (x.l != y.l ? x.l < y.l : x.p < y.p);
            });
            // incidence CSR over the tile's columns (offsets into the global list)
            std::vector<int64_t> counts((size_t)nsel + 1, 0);
            for (const Trip& t : trip) ++counts[(size_t)t.c + 1];
            int64_t acc = ninc;
            for (int64_t c = 0; c <= nsel; ++c) {
                acc += counts[(size_t)c];
                b->inc_ptr.push_back((int32_t)acc);
            }
            for (int64_t r0 = 0; r0 < nr; r0 += kTile) {
                const int64_t r1 = std::min(nr, r0 + kTile);
                b->jobs.insert(b->jobs.end(), {nrow, r1 - r0, npan, np, c0, nsel, out_off[bk] + r0 * ld[bk] + c0, ld[bk]});
                for (int64_t r = r0; r < r1; ++r) b->row_idx.push_back((int32_t)R[r]);
                nrow += r1 - r0;
                b->inc_base.push_back(nptr);
            }
            for (int64_t p : pans) b->pan_idx.push_back((int32_t)p);
            npan += np;
            nptr += nsel + 1;
            for (const Trip& t : trip) b->inc.push_back((t.p << 2) | t.l);
            ninc += (int64_t)trip.size();
            c0 = c1;
        }
    }
    return H2B_OK;
}
}  // namespace

extern "C" int h2b_dlp_jobs_build(int64_t n_verts, const int64_t* vptr, const int64_t* vidx, const int64_t* tris,
                                  int64_t n_blocks, const int64_t* row_ptr, const int64_t* rows,
                                  const int64_t* col_ptr, const int64_t* cols, const int64_t* out_off,
                                  const int64_t* ld, h2b_dlp_build** out) {
    if (!out || (n_blocks > 0 && (!vptr || !vidx || !tris || !row_ptr || !rows || !col_ptr || !cols || !out_off || !ld)))
        return fail(H2B_ERR_INVALID, "h2b_dlp_jobs_build: null pointer");
    h2b_dlp_build* b = new (std::nothrow) h2b_dlp_build();
    if (!b) return fail(H2B_ERR_INVALID, "h2b_dlp_jobs_build: out of host memory");
    // block ranges built in parallel (independent), then concatenated in block
    // order with the offsets shifted: identical to one sequential pass
    const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency());
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hw, n_blocks / 256));
    std::vector<h2b_dlp_build> part((size_t)nt);
    std::vector<int> rc((size_t)nt, H2B_OK);
    std::vector<std::string> err((size_t)nt);
    {
        std::vector<std::thread> th;
        for (int64_t t = 0; t < nt; ++t) {
            const int64_t b0 = n_blocks * t / nt, b1 = n_blocks * (t + 1) / nt;
            auto job = [&, t, b0, b1] {
                rc[(size_t)t] = build_range(n_verts, vptr, vidx, tris, b0, b1, row_ptr, rows, col_ptr, cols, out_off,
                                            ld, &part[(size_t)t], err[(size_t)t]);
            };
            if (nt == 1)
                job();
            else
                th.emplace_back(job);
        }
        for (auto& x : th) x.join();
    }
    for (int64_t t = 0; t < nt; ++t)
        if (rc[(size_t)t] != H2B_OK) {
            delete b;
            return fail(rc[(size_t)t], err[(size_t)t]);
        }
    int64_t nrow = 0, npan = 0, ninc = 0, nptr = 0;
    for (int64_t t = 0; t < nt; ++t) {
        const h2b_dlp_build& q = part[(size_t)t];
        for (size_t j = 0; j < q.jobs.size(); j += 8) {
            b->jobs.insert(b->jobs.end(), q.jobs.begin() + j, q.jobs.begin() + j + 8);
            b->jobs[b->jobs.size() - 8] += nrow;
            b->jobs[b->jobs.size() - 6] += npan;
        }
        for (int32_t v : q.inc_ptr) b->inc_ptr.push_back((int32_t)(v + ninc));
        for (int64_t v : q.inc_base) b->inc_base.push_back(v + nptr);
        b->row_idx.insert(b->row_idx.end(), q.row_idx.begin(), q.row_idx.end());
        b->pan_idx.insert(b->pan_idx.end(), q.pan_idx.begin(), q.pan_idx.end());
        b->inc.insert(b->inc.end(), q.inc.begin(), q.inc.end());
        nrow += (int64_t)q.row_idx.size();
        npan += (int64_t)q.pan_idx.size();
        ninc += (int64_t)q.inc.size();
        nptr += (int64_t)q.inc_ptr.size();
    }
    *out = b;
    return ok();
}

// sizes: jobs (count), row_idx, pan_idx, inc_ptr, inc, inc_base (elements)
extern "C" int h2b_dlp_jobs_sizes(const h2b_dlp_build* b, int64_t* sizes) {
    if (!b || !sizes) return fail(H2B_ERR_INVALID, "h2b_dlp_jobs_sizes: null pointer");
    sizes[0] = (int64_t)b->jobs.size() / 8;
    sizes[1] = (int64_t)b->row_idx.size();
    sizes[2] = (int64_t)b->pan_idx.size();
    sizes[3] = (int64_t)b->inc_ptr.size();
    sizes[4] = (int64_t)b->inc.size();
    sizes[5] = (int64_t)b->inc_base.size();
    return ok();
}

extern "C" int h2b_dlp_jobs_copy(const h2b_dlp_build* b, int64_t* jobs, int32_t* row_idx, int32_t* pan_idx,
                                 int32_t* inc_ptr, int32_t* inc, int64_t* inc_base) {
    if (!b) return fail(H2B_ERR_INVALID, "h2b_dlp_jobs_copy: null pointer");
    auto put = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    put(jobs, b->jobs);
    put(row_idx, b->row_idx);
    put(pan_idx, b->pan_idx);
    put(inc_ptr, b->inc_ptr);
    put(inc, b->inc);
    put(inc_base, b->inc_base);
    return ok();
}

extern "C" int h2b_dlp_jobs_free(h2b_dlp_build* b) {
    delete b;
    return ok();
}
