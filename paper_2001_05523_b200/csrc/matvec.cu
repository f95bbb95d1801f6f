// H^2-matrix-vector product y = A x (containers.py:254-270) in ONE launch.
//
// Work is cut into CTA-sized tasks; every CTA takes a ticket (atomic counter)
// that selects its task.  A task only ever waits for data produced by tasks
// with smaller tickets that never wait on larger ones, so the launch cannot
// deadlock for any grid size or residency.
//
// Inter-CTA data travel in "LL" (low-latency) form: every double is stored as
// two 8-byte units (32-bit payload | 32-bit launch epoch).  An 8-byte access
// is single-copy atomic, so a reader that sees the current epoch in both units
// has the value: data and flag arrive in the same transaction, with no
// fences, no separate flag round trip and nothing to reset between launches
// (the epoch advances every launch).  This is the idea of NCCL's LL protocol,
// applied to the tree transforms.
//
// Every task starts from a host-built record (plan creation), so its first
// memory round trip already yields all offsets it needs:
//
//   A forward   tickets [0, c_leaves) in leaf preorder: x_hat_t = V_t^T x|_t
//               (V_t by TMA bulk copy, x gathered through col_perm).  Then the
//               CTA climbs while its cluster is the RIGHT child: it reads the
//               left sibling's coefficients (written by a smaller ticket),
//               computes x_hat_p = E_c0^T x_hat_c0 + E_c1^T x_hat_c1
//               (ClusterBasis.forward, containers.py:201-212; [E_c0; E_c1]
//               staged by cp.async while it waits) and publishes x_hat_p.
//   B near      one band of rows of a row leaf's nearfield matrix
//               [D_b1 D_b2 ...] (contiguous in HBM; one TMA bulk copy lands
//               while the right-hand side is gathered): y_near = D x|_cols
//               (containers.py:266-267).  Never waits.
//   C coupling  one band of rows of a row cluster's coupling matrix
//               [S_b1 S_b2 ...] (TMA): y_cpl = S [x_hat_s ...]
//               (containers.py:259-264), reading the x_hat in LL form.
//               Bands are ticketed parents first; the LAST band of cluster t
//               (an empty band if t has no couplings) also runs t's downward
//               step v_t = y_cpl_t + E_t v_parent (ClusterBasis.backward,
//               containers.py:214-228): inner clusters publish v_t, leaves
//               write y[row_perm] = y_near + V_t v_t (containers.py:268-269).
//               The downward chain thus advances while the remaining
//               coupling bands stream.
//
// Every output value is produced by one warp or thread in a fixed order:
// bitwise reproducible, no atomics on values, and independent of the number
// of GPUs (row sharding keeps per-row order).  The last CTA to finish resets
// the ticket counter and advances the epoch, so the launch is self-contained
// and can be captured in a CUDA graph.

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <unistd.h>
#include <vector>

#include "device_common.cuh"
#include "nccl_api.h"

namespace h2b {
namespace {

#ifndef H2B_THREADS
#define H2B_THREADS 128
#endif
constexpr int kThreads = H2B_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxVec = 512;        // max rank / leaf size of the vectors kept in smem
constexpr int kMaxDepth = 32;
// TMA staging buffer per CTA (one band): chosen per plan at creation
// (plan_stage_bytes) from the shared memory the rest of the CTA needs
constexpr int kStageMin = 16 * 1024, kStageMax = 40 * 1024;

// record layouts (int64 words)
constexpr int kBandWords = 24;  // src_off, cols, rows, gidx_off, out_off, is_last, has_cpl, kind, then the
                                // downward-step record of the band's cluster (coupling bands):
                                // k, parent y_hat offset (-1 root), k_parent, e_off, y_hat offset,
                                // is_leaf, v_off, start (size = rows of a leaf)
constexpr int kFwdHead = 8;     // start, size, k, v_off, xhat_off, n_climb, warp_ok, offset of the climb levels
constexpr int kFwdStride = 40;  // forward records are fixed-stride (record = ticket * stride: no index round
                                // trip): the header, then the leaf's first 64 x indices (col_perm, int32)
constexpr int kFwdLevel = 6;    // k0, kp, e_off_c0, e_off_own, xhat_off_c0, xhat_off_parent
constexpr int kKindNear = 0, kKindCpl = 1;  // band record kinds (word 7)
constexpr int kFwdAhead = 2048;              // forward tasks pull the record of the task this many tickets on into L2
constexpr int64_t kUpfrontMax = 24 << 20;   // records + gather lists prefetched up front when at most this many bytes
// symmetric nearfield band (see task_panel): words 8..10 = offset of the
// transposed outputs (column c -> 8 + c), leading diagonal-block columns
// without a transposed output, gather offset of the row leaf's own x
constexpr int kKindNearSym = 4;

}  // namespace
}  // namespace h2b

struct h2b_plan {
    h2b_layout L;
    int device;
    uint64_t* xhat;     // LL: 2 x xhat_len
    uint64_t* ycpl;     // LL: 2 x yhat_len (coupling part of y_hat)
    uint64_t* yfin;     // LL: 2 x yhat_len (final y_hat of inner clusters)
    uint64_t* ynear;    // LL: 2 x n_rows (permuted order)
    unsigned long long* ctrl;  // ticket counters ([0] matvec launches, [3] x_hat forward launches), monotonic over launches
    int64_t* rec;       // task records
    int64_t* fwd_off;   // per column leaf: record offset
    int64_t band_base;  // record offset of band 0
    int64_t dgidx_bytes;
    int n_near, n_cpl;
    int max_cols, vec_len;
    int smem;
    int stage_bytes;     // TMA staging buffer per CTA (plan_stage_bytes)
    int64_t e_bytes_r;
    double* dpack = nullptr;  // downward-step operands [E_t^T | V_t^T] per cluster (k_pack_descent)
    double* dx;
    double* dy;
    double* hx = nullptr;  // page-locked staging of a pageable host x (h2b_matvec_host)
    unsigned long long* trace;  // optional per-CTA timeline (H2B_TRACE=1)
    // symmetric nearfield (one copy of every block pair; null when unused)
    double* dsym;       // packed column panels of the upper blocks
    int32_t* gsym;      // their gather indices
    uint64_t* ppart;    // LL partial vectors (direct per panel, transposed per block)
    int64_t* nsum;      // per leaf: the partials summed by its final task, in order
    int64_t ppart_len;
    int64_t near_bytes; // nearfield bytes one matvec streams
    int64_t cpl_bytes;  // coupling bytes one matvec streams
    // Launches of one plan must run one after another (one ticket counter and
    // one set of LL scratch buffers per plan): a host mutex serialises callers,
    // and a launch on a different stream than the previous one first waits
    // for it (event), so stream-ordered use from any stream is safe.
    std::mutex mu;
    cudaEvent_t done = nullptr;
    cudaStream_t last = nullptr;
    bool launched = false;
    // x_hat exchange (h2b_plan_create_xhat): the forward tasks cover only this
    // rank's column clusters (own launch, own LL buffer xhat_f); their
    // coefficients leave through h2b_xhat_forward, everybody's come back in
    // through h2b_xhat_main, which climbs the clusters spanning several ranks
    // and launches the bands with no forward task
    int n_fwd = 0;              // forward tasks per launch
    bool xmode = false;
    uint64_t* xhat_f = nullptr;
    int32_t* d_own = nullptr;   // owned clusters (send order) and their send offsets
    int64_t* d_own_off = nullptr;
    int n_own = 0;
    int64_t send_len = 0;
    int32_t* d_imp = nullptr;   // gathered clusters and their offsets in the gathered buffer
    int64_t* d_imp_src = nullptr;
    int n_imp = 0;
    int32_t* d_span = nullptr;  // spanning clusters, deepest level first
    std::vector<int64_t> span_level_off;
    double* span_val = nullptr; // plain coefficients (x_hat offsets) for the spanning climbs
    unsigned long long n_f_launches = 0, n_m_launches = 0;
    // row sharding over NCCL (h2b_plan_set_comm)
    void* comm = nullptr;
    int comm_rank = 0, comm_size = 1;
    int64_t comm_chunk = 0;
    double* xgath = nullptr;  // comm_size x comm_chunk gathered x
};

namespace h2b {
namespace {

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifdef H2B_LL_TIMEOUT
__device__ unsigned long long g_mbar_stuck[4];  // block + 1, parity, abandoned waits, longest wait (ns)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef H2B_LL_TIMEOUT
    // debug builds: a wait abandoned after 2 s is recorded instead of hanging
    // the GPU, and the longest wait is kept.  (The bound is on time: a bare
    // test_wait loop bounded by an iteration count reported waits that the
    // polling itself had slowed down.)
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (ok) {
            atomicMax(&g_mbar_stuck[3], t1 - t0);
            return;
        }
        if (t1 - t0 > 2000000000ull) {
            g_mbar_stuck[0] = blockIdx.x + 1;
            g_mbar_stuck[1] = parity;
            atomicAdd(&g_mbar_stuck[2], 1ull);
            return;
        }
    }
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D TMA bulk copy global -> shared (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    // operator bytes are read once per matvec: evict-first in L2, so the
    // stream does not push out what is reused (x, x_hat, partials, records);
    // config 1 51.6 -> 49.6 us, larger configurations neutral
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// LDGSTS: 8-byte asynchronous global -> shared copies; a thread can have many
// in flight (no register staging).
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 1-D bulk prefetch into L2 (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}


// ---- LL form: double -> (lo32 | epoch), (hi32 | epoch) ---------------------
__device__ __forceinline__ void ll_store(uint64_t* p, double v, uint32_t epoch) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    const uint64_t e = static_cast<uint64_t>(epoch) << 32;
    const uint64_t u0 = (b & 0xffffffffull) | e, u1 = (b >> 32) | e;
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(u0), "l"(u1) : "memory");
}

__device__ __forceinline__ bool ll_try(const uint64_t* p, uint32_t epoch, double& v) {
    uint64_t u0, u1;
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(u0), "=l"(u1) : "l"(p) : "memory");
    if ((uint32_t)(u0 >> 32) != epoch || (uint32_t)(u1 >> 32) != epoch) return false;
    v = __longlong_as_double(static_cast<long long>((u0 & 0xffffffffull) | (u1 << 32)));
    return true;
}

#ifdef H2B_LL_TIMEOUT
__device__ unsigned long long g_ll_stuck[4];  // debugging: address / epoch of an abandoned wait
#endif
__device__ __forceinline__ double ll_load(const uint64_t* p, uint32_t epoch) {
    double v;
    if (ll_try(p, epoch, v)) return v;
#ifdef H2B_LL_TIMEOUT
    for (long long it = 0; !ll_try(p, epoch, v); ++it) {
        __nanosleep(32);
#ifndef H2B_LL_TIMEOUT_ITERS
#define H2B_LL_TIMEOUT_ITERS (1ll << 22)
#endif
        if (it > H2B_LL_TIMEOUT_ITERS) {
            g_ll_stuck[0] = reinterpret_cast<unsigned long long>(p);
            g_ll_stuck[1] = epoch;
            g_ll_stuck[2] = blockIdx.x;
            g_ll_stuck[3] = *reinterpret_cast<const volatile unsigned long long*>(p);
            return 0.0;
        }
    }
#else
    while (!ll_try(p, epoch, v)) __nanosleep(32);
#endif
    return v;
}

__device__ __forceinline__ void mark(unsigned long long* m, int i) {
    if (m && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        m[i] = t;
    }
}

// ---------------------------------------------------------------------------
// dense building blocks (operands in shared memory unless noted)

#ifndef H2B_ROWBLOCK
#define H2B_ROWBLOCK 4
#endif
constexpr int kRowBlock = H2B_ROWBLOCK;  // rows per warp in rows_dot's many-rows mode
// widest right-hand side gathered at once (multiple of 128: see task_band);
// wider band rows are processed in chunks of it
#ifndef H2B_CHUNK_COLS
#define H2B_CHUNK_COLS 768
#endif
constexpr int kChunkCols = H2B_CHUNK_COLS;

__host__ __device__ constexpr int log2c(int n) { return n <= 1 ? 0 : 1 + log2c(n / 2); }

// Sum over the warp of N per-lane values by recursive halving (N - 1 + 5 -
// log2 N shuffles); lane l ends with the total of value ri(l), whose bit
// (log2 N - 1 - j) is lane bit (4 - j).
template <int N>
__device__ __forceinline__ double warp_sum(double (&a)[N], int lane) {
    int o = 16;
#pragma unroll
    for (int h = N / 2; h >= 1; h >>= 1, o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? a[i] : a[i + h], keep = up ? a[i + h] : a[i];
            a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    double v = a[0];
#pragma unroll
    for (; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One warp: out[r0 + i] = M[(r0 + i) * ld : ...] . v, i < nr <= R.  Lanes
// stride the columns; every lane keeps R independent FMA chains and reads
// v[c] once for all R rows.  Rows past nr re-read the last row (branch-free
// loads, results dropped).
template <int R>
__device__ __forceinline__ void rows_warp(const double* M, int64_t ld, int r0, int nr, int cols, const double* v,
                                          double* out, int lane) {
    if (nr <= 0) return;
    const double* m[R];
#pragma unroll
    for (int i = 0; i < R; ++i) m[i] = M + (int64_t)(r0 + min(i, nr - 1)) * ld;
    double acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = 0.0;
#pragma unroll 4
    for (int c = lane; c < cols; c += 32) {
        const double vc = v[c];
        double e[R];
#pragma unroll
        for (int i = 0; i < R; ++i) e[i] = m[i][c];
#pragma unroll
        for (int i = 0; i < R; ++i) acc[i] = fma(e[i], vc, acc[i]);
    }
    const double sum = warp_sum<R>(acc, lane);
    constexpr int lg = log2c(R), sh = 5 - lg;
    int ri = 0;
#pragma unroll
    for (int j = 0; j < lg; ++j) ri |= ((lane >> (4 - j)) & 1) << (lg - 1 - j);
    if ((lane & ((1 << sh) - 1)) == 0 && ri < nr) out[r0 + ri] = sum;
}

// out[i] = M[i*ld : i*ld+cols] . v, i < rows.  Few rows: one row per warp
// (four partial sums per lane); many rows: each warp owns 4 rows at a time
// (4 independent dot products, interleaved shuffle reductions).
__device__ void rows_dot(const double* M, int64_t ld, int rows, int cols, const double* v,
                                         double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (rows <= kWarps) {
        if (warp < rows) {
            const double* row = M + (int64_t)warp * ld;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int c = lane;
            for (; c + 96 < cols; c += 128) {
                const double m0 = row[c], m1 = row[c + 32], m2 = row[c + 64], m3 = row[c + 96];
                const double v0 = v[c], v1 = v[c + 32], v2 = v[c + 64], v3 = v[c + 96];
                a0 = fma(m0, v0, a0);
                a1 = fma(m1, v1, a1);
                a2 = fma(m2, v2, a2);
                a3 = fma(m3, v3, a3);
            }
            for (; c < cols; c += 32) a0 = fma(row[c], v[c], a0);
            double sum = (a0 + a1) + (a2 + a3);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) out[warp] = sum;
        }
        return;
    }
    if (rows <= 2 * kWarps) {
        rows_warp<2>(M, ld, 2 * warp, min(2, rows - 2 * warp), cols, v, out, lane);
        return;
    }
    for (int r0 = kRowBlock * warp; r0 < rows; r0 += kRowBlock * kWarps)
        rows_warp<kRowBlock>(M, ld, r0, min(kRowBlock, rows - r0), cols, v, out, lane);
}

// out[c] = sum_r M[r*k + c] v[r], c < k: warps split rows, lanes columns,
// partials reduced through `red` (kWarps x 32).  Ends with __syncthreads().
__device__ void cols_dot(const double* M, int rows, int k, const double* v, double* red, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int c = c0 + lane;
        double a0 = 0.0, a1 = 0.0;
        if (c < k) {
            int r = warp;
            for (; r + kWarps < rows; r += 2 * kWarps) {
                a0 = fma(M[(int64_t)r * k + c], v[r], a0);
                a1 = fma(M[(int64_t)(r + kWarps) * k + c], v[r + kWarps], a1);
            }
            if (r < rows) a0 = fma(M[(int64_t)r * k + c], v[r], a0);
        }
        red[warp * 32 + lane] = a0 + a1;
        __syncthreads();
        if (warp == 0 && c < k) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s += red[w * 32 + lane];
            out[c] = s;
        }
        __syncthreads();
    }
}

// Small dense products (transfer matrices, leaf bases: at most a few hundred
// columns), one thread per output: no reductions, no barriers inside; four
// interleaved partial sums per thread; operands in shared or global memory.
// out[r] = M[r*ld : r*ld+cols] . v, r < rows
__device__ __forceinline__ void small_rows_dot(const double* M, int64_t ld, int rows, int cols, const double* v,
                                               double* out) {
    for (int r = threadIdx.x; r < rows; r += kThreads) {
        const double* m = M + (int64_t)r * ld;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = 0;
        for (; c + 3 < cols; c += 4) {
            a0 = fma(m[c], v[c], a0);
            a1 = fma(m[c + 1], v[c + 1], a1);
            a2 = fma(m[c + 2], v[c + 2], a2);
            a3 = fma(m[c + 3], v[c + 3], a3);
        }
        for (; c < cols; ++c) a0 = fma(m[c], v[c], a0);
        out[r] = (a0 + a1) + (a2 + a3);
    }
}

// out[c] = sum_r M[r*k + c] v[r], c < k.  With at most 32 outputs, the warps
// split the rows (interleaved) and the partials are summed in a fixed order
// through red (kWarps x 32): ends with __syncthreads() in that case.
__device__ __forceinline__ void small_cols_dot(const double* M, int rows, int k, const double* v, double* out,
                                               double* red) {
    if (k <= 32 && red) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane < k) {
            double a0 = 0.0, a1 = 0.0;
            int r = warp;
            for (; r + kWarps < rows; r += 2 * kWarps) {
                a0 = fma(M[(int64_t)r * k + lane], v[r], a0);
                a1 = fma(M[(int64_t)(r + kWarps) * k + lane], v[r + kWarps], a1);
            }
            if (r < rows) a0 = fma(M[(int64_t)r * k + lane], v[r], a0);
            red[warp * 32 + lane] = a0 + a1;
        }
        __syncthreads();
        if (warp == 0 && lane < k) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) t += red[w * 32 + lane];
            out[lane] = t;
        }
        __syncthreads();
        return;
    }
    for (int c = threadIdx.x; c < k; c += kThreads) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int r = 0;
        for (; r + 3 < rows; r += 4) {
            a0 = fma(M[(int64_t)r * k + c], v[r], a0);
            a1 = fma(M[(int64_t)(r + 1) * k + c], v[r + 1], a1);
            a2 = fma(M[(int64_t)(r + 2) * k + c], v[r + 2], a2);
            a3 = fma(M[(int64_t)(r + 3) * k + c], v[r + 3], a3);
        }
        for (; r < rows; ++r) a0 = fma(M[(int64_t)r * k + c], v[r], a0);
        out[c] = (a0 + a1) + (a2 + a3);
    }
}

// Gather rhs[i] = src[idx[i]], i < n: all index loads, then all value loads.
__device__ __forceinline__ void gather(double* rhs, const double* __restrict__ src, const int32_t* idx, int n) {
    constexpr int kU = 4;
    for (int base = 0; base < n; base += kU * kThreads) {
        int ix[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = base + u * kThreads + (int)threadIdx.x;
            ix[u] = i < n ? __ldg(idx + i) : -1;
        }
        double v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = ix[u] >= 0 ? __ldg(src + ix[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = base + u * kThreads + (int)threadIdx.x;
            if (i < n) rhs[i] = v[u];
        }
    }
}

// Gather from LL form: rhs[i] = LL[idx[i]] (spins until the producer's epoch).
// (all index loads, then all LL loads in flight at once; spin only on the
// entries whose producer has not published yet)
__device__ __forceinline__ void gather_ll(double* rhs, const uint64_t* ll, const int32_t* idx, int n,
                                          uint32_t epoch) {
    uint64_t pol_el;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_el));
    constexpr int kU = 1024 / kThreads;
    for (int base = 0; base < n; base += kU * kThreads) {
        int ix[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = base + u * kThreads + (int)threadIdx.x;
            ix[u] = i < n ? __ldg(idx + i) : -1;
        }
        uint64_t w0[kU], w1[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            w0[u] = w1[u] = 0;
            if (ix[u] >= 0)
                asm volatile("ld.relaxed.gpu.global.L2::cache_hint.v2.b64 {%0, %1}, [%2], %3;"
                             : "=l"(w0[u]), "=l"(w1[u])
                             : "l"(ll + 2 * (int64_t)ix[u]), "l"(pol_el));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (ix[u] < 0) continue;
            double v;
            if ((uint32_t)(w0[u] >> 32) == epoch && (uint32_t)(w1[u] >> 32) == epoch)
                v = __longlong_as_double(static_cast<long long>((w0[u] & 0xffffffffull) | (w1[u] << 32)));
            else
                v = ll_load(ll + 2 * (int64_t)ix[u], epoch);
            rhs[base + u * kThreads + (int)threadIdx.x] = v;
        }
    }
}

struct Shared {
    unsigned long long* mark;  // trace slots of this CTA (5 phase marks) or null
    uint64_t* bar;             // mbarrier of the staging buffer
    char* stage;               // stage_bytes, 128-byte aligned
    int stage_bytes;           // the plan's staging buffer size
    double* rhs;               // max_cols
    double* va;                // 2 vec_len ([x_hat_c0; x_hat_c1] in the climb)
    double* vb;                // vec_len (vec_len = max rank / leaf size)
    double* red;               // kWarps * 64
    int64_t* rec;              // small record cache
    const int64_t* rec_src;    // the forward task's record in global memory
    double* yn;                // vec_len: a leaf's summed nearfield rows (symmetric nearfield)
    const uint64_t* ppart;     // symmetric nearfield partials or null
    const int64_t* nsum;       // their per-leaf lists
    bool near_sym;             // nearfield as symmetric column panels
    uint32_t parity;           // mbarrier phase of the staging slot in use
    const double* dpack;       // downward-step operands [E_t^T | V_t^T] per cluster (plan-owned copy)
    int64_t pf;                // this thread's partial vector to pull into L2 (leaf final tasks), or -1
};


// Thread 0 starts staging `bytes` (TMA bulk copy when it fits and is 16-byte
// aligned; otherwise a plain arrive).  Returns where to read the data from.
__device__ __forceinline__ const double* stage_issue(const Shared& s, const double* src, int64_t bytes) {
    const bool fits = bytes > 0 && bytes <= s.stage_bytes && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                      (bytes & 15) == 0;
    if (threadIdx.x == 0) {
        if (fits) {
            mbar_expect_tx(s.bar, (uint32_t)bytes);
            bulk_g2s(s.stage, src, (uint32_t)bytes, s.bar);
        } else {
            mbar_arrive(s.bar);
        }
    }
    return fits ? reinterpret_cast<const double*>(s.stage) : src;
}

__device__ void prefetch_slice(const double* base, int64_t bytes, int part, int parts) {
    if (!base || bytes <= 0) return;
    const int64_t lines = (bytes + 127) / 128;
    const int64_t per = (lines + parts - 1) / parts;
    const int64_t l0 = per * part, l1 = min(lines, l0 + per);
    const char* b = reinterpret_cast<const char*>(base);
    for (int64_t l = l0 + threadIdx.x; l < l1; l += blockDim.x) prefetch_l2(b + 128 * l);
}

// copy a record of n words into the shared record cache (one round trip)
__device__ __forceinline__ void load_rec(const Shared& s, const int64_t* src, int n) {
    for (int i = threadIdx.x; i < n; i += kThreads) s.rec[i] = __ldg(src + i);
    __syncthreads();
}

// The forward products of a warp (lane c owns coefficient c, ranks <= 32), in
// ONE summation order whichever task path runs them (a task takes the
// one-warp path only when its whole climb fits; the value of a coefficient must
// not depend on that, so row sharding -- which shortens climbs -- keeps the
// single-GPU bits).  Leaf: x_hat[c] = sum_r V[r, c] x[r] (even / odd rows in
// two chains); climb: x_hat_p[c] = E_c0^T x_hat_c0 + E_c1^T x_hat_c1 (two
// chains each).
__device__ __forceinline__ double leaf_coef(const double* V, int size, int k, const double* xv, int lane) {
    double a0 = 0.0, a1 = 0.0;
    int r = 0;
    for (; r + 1 < size; r += 2) {
        a0 = fma(V[(int64_t)r * k + lane], xv[r], a0);
        a1 = fma(V[(int64_t)(r + 1) * k + lane], xv[r + 1], a1);
    }
    if (r < size) a0 = fma(V[(int64_t)r * k + lane], xv[r], a0);
    return a0 + a1;
}

__device__ __forceinline__ double climb_coef(const double* E0, const double* E1, int k0, int k1, int kp,
                                             const double* v, int lane) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int r = 0;
    for (; r + 1 < k0; r += 2) {
        a0 = fma(E0[r * kp + lane], v[r], a0);
        a1 = fma(E0[(r + 1) * kp + lane], v[r + 1], a1);
    }
    if (r < k0) a0 = fma(E0[r * kp + lane], v[r], a0);
    r = 0;
    for (; r + 1 < k1; r += 2) {
        a2 = fma(E1[r * kp + lane], v[k0 + r], a2);
        a3 = fma(E1[(r + 1) * kp + lane], v[k0 + r + 1], a3);
    }
    if (r < k1) a2 = fma(E1[r * kp + lane], v[k0 + r], a2);
    return (a0 + a1) + (a2 + a3);
}

// Forward task on one warp (chain latency: no block barriers).  Lane c owns
// output coefficient c (ranks <= 32), the leaf has <= 64 rows; operands in
// shared memory, the climb's transfer matrices copied by the warp (cp.async)
// while the sibling's coefficients are awaited.
__device__ void forward_warp(const double* __restrict__ c_V, const double* __restrict__ c_E,
                             const double* __restrict__ x, uint64_t* xhat, uint32_t epoch, const Shared& s,
                             int ix0, int ix1) {
    const int lane = threadIdx.x;
    const int size = (int)s.rec[1], k = (int)s.rec[2];
    const int64_t v_off = s.rec[3], xhat_off = s.rec[4];
    const int n_climb = (int)s.rec[5];
    const double* V = stage_issue(s, c_V + v_off, ((int64_t)size * k * 8 + 15) & ~int64_t(15));
    // x through the permutation: the indices came with the record (ix0, ix1:
    // rows lane and lane + 32), so the values are one round trip away
    if (lane < size) s.va[lane] = __ldg(x + ix0);
    if (lane + 32 < size) s.va[lane + 32] = __ldg(x + ix1);
    for (int i = lane; i < kFwdLevel * n_climb; i += 32) s.rec[kFwdHead + i] = __ldg(s.rec_src + i);
    __syncwarp();
    {
        int kk = k;  // pull the climb's transfer matrices into L2
        for (int j = 0; j < n_climb; ++j) {
            const int64_t* lv = s.rec + kFwdHead + kFwdLevel * j;
            const int kp = (int)lv[1];
            const int64_t b0 = 8 * (int64_t)lv[0] * kp, b1 = 8 * (int64_t)kk * kp;
            const char* e0 = reinterpret_cast<const char*>(c_E + lv[2]);
            const char* e1 = reinterpret_cast<const char*>(c_E + lv[3]);
            for (int64_t o = 128 * lane; o < b0; o += 128 * 32) prefetch_l2(e0 + o);
            for (int64_t o = 128 * lane; o < b1; o += 128 * 32) prefetch_l2(e1 + o);
            kk = kp;
        }
    }
    mbar_wait(s.bar, s.parity);
    double own = 0.0;
    if (lane < k) {
        own = leaf_coef(V, size, k, s.va, lane);
        ll_store(xhat + 2 * (xhat_off + lane), own, epoch);
    }
    mark(s.mark, 0);
    double* buf = reinterpret_cast<double*>(s.stage);
    uint32_t par = s.parity ^ 1u;  // the staging barrier's next phase (V used one)
    int k1 = k;
    for (int j = 0; j < n_climb; ++j) {
        const int64_t* lv = s.rec + kFwdHead + kFwdLevel * j;
        const int k0 = (int)lv[0], kp = (int)lv[1];
        // E_c0 and E_own by two TMA bulk copies (blocks are 16-byte aligned and
        // padded to an even length; the warp path is taken only when both fit)
        const int p0 = (k0 * kp + 1) & ~1, p1 = (k1 * kp + 1) & ~1;
        __syncwarp();  // buf / va free
        if (lane == 0) {
            mbar_expect_tx(s.bar, (uint32_t)(8 * (p0 + p1)));
            bulk_g2s(buf, c_E + lv[2], (uint32_t)(8 * p0), s.bar);
            bulk_g2s(buf + p0, c_E + lv[3], (uint32_t)(8 * p1), s.bar);
        }
        if (lane < k1) s.va[k0 + lane] = own;
        if (lane < k0) s.va[lane] = ll_load(xhat + 2 * (lv[4] + lane), epoch);
        mbar_wait(s.bar, par);
        par ^= 1u;
        __syncwarp();
        if (j < 2) mark(s.mark, 1 + 2 * j);
        own = 0.0;
        if (lane < kp) {
            own = climb_coef(buf, buf + p0, k0, k1, kp, s.va, lane);
            ll_store(xhat + 2 * (lv[5] + lane), own, epoch);
        }
        if (j < 2) mark(s.mark, 2 + 2 * j);
        k1 = kp;
    }
}

// ---------------------------------------------------------------------------
// A: forward transform of one column leaf; climb while the right child

__device__ void task_forward(const double* __restrict__ c_V, const double* __restrict__ c_E,
                                       const int64_t* __restrict__ col_perm, const int64_t* rec, const double* __restrict__ x,
                             uint64_t* xhat, uint32_t epoch, const Shared& s, const int64_t* rec_base) {
    // header and the leaf's x indices in one round trip, then (block path) the
    // climb levels
    int ix0 = 0, ix1 = 0;
    if (threadIdx.x < 32) {
        const int32_t* ip = reinterpret_cast<const int32_t*>(rec + kFwdHead);
        ix0 = __ldg(ip + threadIdx.x);
        ix1 = __ldg(ip + 32 + threadIdx.x);
    }
    for (int i = threadIdx.x; i < kFwdHead; i += kThreads) s.rec[i] = __ldg(rec + i);
    __syncthreads();
    const_cast<Shared&>(s).rec_src = rec_base + s.rec[7];  // the climb levels
    if (!s.rec[6]) {
        const int nc = (int)s.rec[5];
        for (int i = threadIdx.x; i < kFwdLevel * nc; i += kThreads) s.rec[kFwdHead + i] = __ldg(s.rec_src + i);
    }
    const int start = (int)s.rec[0], size = (int)s.rec[1], k = (int)s.rec[2];
    const int64_t v_off = s.rec[3], xhat_off = s.rec[4];
    const int n_climb = (int)s.rec[5];
    if (s.rec[6]) {  // every rank <= 32 and the leaf <= 64 rows: one warp, no block barriers
        if (threadIdx.x < 32) forward_warp(c_V, c_E, x, xhat, epoch, s, ix0, ix1);
        return;
    }
    const double* V = stage_issue(s, c_V + v_off, ((int64_t)size * k * 8 + 15) & ~int64_t(15));
    for (int r = threadIdx.x; r < size; r += blockDim.x) s.va[r] = __ldg(x + col_perm[start + r]);
    mbar_wait(s.bar, s.parity);
    __syncthreads();  // (also: the climb levels are in s.rec)
    {
        // pull every climb level's [E_c0; E_own] into L2 now (the copies into
        // shared memory at each level then hit L2)
        int kk = k;
        for (int j = 0; j < n_climb; ++j) {
            const int64_t* lv = s.rec + kFwdHead + kFwdLevel * j;
            const int kp = (int)lv[1];
            const int64_t b0 = 8 * (int64_t)lv[0] * kp, b1 = 8 * (int64_t)kk * kp;
            const char* e0 = reinterpret_cast<const char*>(c_E + lv[2]);
            const char* e1 = reinterpret_cast<const char*>(c_E + lv[3]);
            for (int64_t o = 128 * threadIdx.x; o < b0; o += 128 * kThreads) prefetch_l2(e0 + o);
            for (int64_t o = 128 * threadIdx.x; o < b1; o += 128 * kThreads) prefetch_l2(e1 + o);
            kk = kp;
        }
    }
    if (k <= 32) {  // the one-warp order (see leaf_coef)
        if (threadIdx.x < k) s.vb[threadIdx.x] = leaf_coef(V, size, k, s.va, threadIdx.x);
    } else {
        small_cols_dot(V, size, k, s.va, s.vb, s.red);  // own coefficients stay in s.vb
    }
    __syncthreads();
    mark(s.mark, 0);
    {
        uint64_t* dst = xhat + 2 * xhat_off;
        for (int c = threadIdx.x; c < k; c += blockDim.x) ll_store(dst + 2 * c, s.vb[c], epoch);
    }
    double* buf = reinterpret_cast<double*>(s.stage);  // [E_c0; E_own]
    int k1 = k;
    for (int j = 0; j < n_climb; ++j) {
        const int64_t* lv = s.rec + kFwdHead + kFwdLevel * j;
        const int k0 = (int)lv[0], kp = (int)lv[1];
        const int n0 = k0 * kp, n1 = k1 * kp;
        const bool in_smem = (n0 + n1) * 8 <= s.stage_bytes;
        __syncthreads();  // previous users of buf / va are done
        if (in_smem) {
            const double* E0 = c_E + lv[2];
            const double* E1 = c_E + lv[3];
            for (int i = threadIdx.x; i < n0; i += kThreads) cp_async8(buf + i, E0 + i);
            for (int i = threadIdx.x; i < n1; i += kThreads) cp_async8(buf + n0 + i, E1 + i);
        }
        // v = [x_hat_c0; x_hat_own]: the left sibling's from LL (smaller ticket)
        const uint64_t* xs = xhat + 2 * lv[4];
        for (int r = threadIdx.x; r < k0; r += kThreads) s.va[r] = ll_load(xs + 2 * r, epoch);
        for (int r = threadIdx.x; r < k1; r += kThreads) s.va[k0 + r] = s.vb[r];
        cp_async_wait_all();
        __syncthreads();
        if (j < 2) mark(s.mark, 1 + 2 * j);
        if (in_smem && kp <= 32) {  // the one-warp order (see climb_coef)
            if (threadIdx.x < kp) s.vb[threadIdx.x] = climb_coef(buf, buf + n0, k0, k1, kp, s.va, threadIdx.x);
            __syncthreads();
        } else if (in_smem) {
            small_cols_dot(buf, k0 + k1, kp, s.va, s.vb, s.red);
            __syncthreads();
        } else {
            cols_dot(c_E + lv[2], k0, kp, s.va, s.red, s.vb);
            for (int c = threadIdx.x; c < kp; c += kThreads) s.rhs[c] = s.vb[c];
            __syncthreads();
            cols_dot(c_E + lv[3], k1, kp, s.va + k0, s.red, s.vb);
            for (int c = threadIdx.x; c < kp; c += kThreads) s.vb[c] += s.rhs[c];
            __syncthreads();
        }
        uint64_t* dst = xhat + 2 * lv[5];
        for (int c = threadIdx.x; c < kp; c += kThreads) ll_store(dst + 2 * c, s.vb[c], epoch);
        if (j < 2) mark(s.mark, 2 + 2 * j);
        k1 = kp;
    }
}

// ---------------------------------------------------------------------------
// B / C: one band of a nearfield (x gathered) or coupling (x_hat, LL) matrix

// Downward step of a row cluster t, run by the last coupling band of t (or by
// an empty band when t has no couplings):  v_t = y_cpl_t + E_t v_parent
// (ClusterBasis.backward, containers.py:214-228).  Inner clusters publish v_t
// (LL); a leaf expands y[row_perm] = y_near + V_t v_t (containers.py:268-269).
// Every value waited for is produced by a smaller ticket: the other bands of
// t, the parent's last band (parents are ticketed first) and the near bands.
// Symmetric nearfield: s.yn[i] = sum of the n partial vectors listed at
// `list` (LL offsets into s.ppart), i < size, always in list order.  H threads
// per row take contiguous parts of the list (their sums are added in part
// order); each thread keeps 8 loads in flight.  Ends with a block barrier.
// Threads [t0, t0 + nt) take part; bar_id 0 = block barrier, else a named
// barrier over those nt threads.
__device__ void near_sum(const Shared& s, const int64_t* list, int n, int size, uint32_t epoch, double* out,
                         int t0 = 0, int nt = kThreads, int bar_id = 0) {
    int H = 1;
    while (H < 4 && 2 * H * size <= nt) H *= 2;
    const int tid = (int)threadIdx.x - t0;
    const int step = H == 1 ? nt : size;
    for (int base = 0; base < size; base += step) {
        const int h = H == 1 ? 0 : tid / size;
        const int i = base + (H == 1 ? tid : tid - h * size);
        double acc = 0.0;
        if (h < H && i < size) {
            const int m0 = (n * h) / H, m1 = (n * (h + 1)) / H;
            for (int m = m0; m < m1; m += 8) {
                uint64_t w0[8], w1[8];
                const uint64_t* src[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    src[u] = m + u < m1 ? s.ppart + 2 * (__ldg(list + m + u) + i) : nullptr;
                    w0[u] = w1[u] = 0;
                    if (src[u])
                        asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                                     : "=l"(w0[u]), "=l"(w1[u])
                                     : "l"(src[u]));
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (!src[u]) continue;
                    double v;
                    if ((uint32_t)(w0[u] >> 32) == epoch && (uint32_t)(w1[u] >> 32) == epoch)
                        v = __longlong_as_double(static_cast<long long>((w0[u] & 0xffffffffull) | (w1[u] << 32)));
                    else
                        v = ll_load(src[u], epoch);
                    acc += v;
                }
            }
        }
        if (H == 1) {
            if (i < size) out[i] = acc;
        } else if (h < H && i < size) {
            s.red[h * size + i] = acc;
        }
    }
    auto sync = [&]() {
        if (bar_id == 0)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nt) : "memory");
    };
    sync();
    if (H > 1) {
        for (int i = tid; i < size; i += nt) {
            double t = 0.0;
            for (int h = 0; h < H; ++h) t += s.red[h * size + i];
            out[i] = t;
        }
        sync();
    }
}

// `par`: the staging barrier's next phase.  The operands come from the plan's
// packed copy s.dpack: per cluster E_t^T (k_parent x k, padded to an even
// length) followed by V_t^T (k x |t|, leaves), so ONE bulk copy stages what
// the thread-per-row products read (the one-warp step used to transpose both
// with 8-byte cp.async copies: ~5 us of a 10 us leaf task at config 3).
__device__ void descent(const double* __restrict__ r_E, const double* __restrict__ r_V,
                                  const int64_t* __restrict__ row_perm, const int64_t* d, const uint64_t* ycpl, uint64_t* yfin,
                        const uint64_t* ynear, double* y, uint32_t epoch, bool has_cpl, const Shared& s, uint32_t par) {
    const int k = (int)d[0], kp = (int)d[2];
    const int64_t par_off = d[1], e_off = d[3], yoff = d[4];
    const bool leaf = d[5] != 0;
    const int64_t v_off = d[6];
    const int start = (int)d[7];
    double* Es = reinterpret_cast<double*>(s.stage);
    // symmetric nearfield: this leaf's rows are the sum of its partials
    const bool sym = leaf && s.near_sym && d[12] > 0;
    // (one-warp downward step: warps 1..3 sum the partials meanwhile, below)
    if (sym && !d[10]) near_sum(s, s.nsum + d[11], (int)d[12], (int)d[8], epoch, s.yn);
    if (d[10]) {  // (record word 18) ranks <= 32, leaf <= 64 rows: one warp, no block barriers
        if (threadIdx.x >= 32) {
            if (sym) {
                // the leaf's nearfield rows, while warp 0 waits for its inputs;
                // named barrier 2 (all 128 threads) hands s.yn over to warp 0
                near_sum(s, s.nsum + d[11], (int)d[12], (int)d[8], epoch, s.yn, 32, kThreads - 32, 1);
                asm volatile("bar.sync 2, %0;" ::"r"(kThreads) : "memory");
            }
            return;
        }
        const int lane = threadIdx.x;
        const int size = leaf ? (int)d[8] : 0;
        double* Vt = Es + ((k * kp + 1) & ~1);
        // [E_t^T | V_t^T] by one bulk copy while the inputs are awaited
        const uint32_t pbytes = 8u * (uint32_t)(((k * kp + 1) & ~1) + ((size * k + 1) & ~1));
        if (pbytes && lane == 0) {
            mbar_expect_tx(s.bar, pbytes);
            bulk_g2s(Es, s.dpack + d[13], pbytes, s.bar);
        }
        // (the rows' output indices now: their latency would sit at the very end of the task)
        int64_t rp0 = 0, rp1 = 0;
        if (leaf && lane < size) rp0 = __ldg(row_perm + start + lane);
        if (leaf && lane + 32 < size) rp1 = __ldg(row_perm + start + lane + 32);
        double v = (has_cpl && lane < k) ? ll_load(ycpl + 2 * (yoff + lane), epoch) : 0.0;
        if (par_off >= 0 && lane < kp) s.rhs[lane] = ll_load(yfin + 2 * (par_off + lane), epoch);
        if (pbytes) mbar_wait(s.bar, par);
        __syncwarp();
        mark(s.mark, 4);
        if (par_off >= 0 && lane < k) {
            double a0 = 0.0, a1 = 0.0;
            int c = 0;
            for (; c + 1 < kp; c += 2) {
                a0 = fma(Es[c * k + lane], s.rhs[c], a0);
                a1 = fma(Es[(c + 1) * k + lane], s.rhs[c + 1], a1);
            }
            if (c < kp) a0 = fma(Es[c * k + lane], s.rhs[c], a0);
            v += a0 + a1;
        }
        mark(s.mark, 1);
        if (!leaf) {
            if (lane < k) ll_store(yfin + 2 * (yoff + lane), v, epoch);
            return;
        }
        if (lane < k) s.vb[lane] = v;
        if (sym)
            asm volatile("bar.sync 2, %0;" ::"r"(kThreads) : "memory");  // s.yn from warps 1..3
        else
            __syncwarp();
        for (int i = lane; i < size; i += 32) {
            double a0 = 0.0, a1 = 0.0;
            int r = 0;
            for (; r + 1 < k; r += 2) {
                a0 = fma(Vt[r * size + i], s.vb[r], a0);
                a1 = fma(Vt[(r + 1) * size + i], s.vb[r + 1], a1);
            }
            if (r < k) a0 = fma(Vt[r * size + i], s.vb[r], a0);
            y[i < 32 ? rp0 : rp1] =
                (sym ? s.yn[i] : ll_load(ynear + 2 * ((int64_t)start + i), epoch)) + (a0 + a1);
        }
        return;
    }
    const int ne = (k * kp + 1) & ~1;  // E_t^T in the packed copy (padded to an even length)
    const bool e_smem = par_off >= 0 && k > 0 && ne <= s.stage_bytes / 8;
    // transfer / leaf basis matrices are staged TRANSPOSED (the packed copy
    // holds them so), so that the thread-per-row products below read
    // consecutive words (no bank conflicts)
    if (e_smem && threadIdx.x == 0) {
        mbar_expect_tx(s.bar, 8u * (uint32_t)ne);
        bulk_g2s(Es, s.dpack + d[13], 8u * (uint32_t)ne, s.bar);
    }
    const uint64_t* yc = ycpl + 2 * yoff;
    for (int i = threadIdx.x; i < k; i += kThreads)
        s.va[i] = has_cpl ? ll_load(yc + 2 * i, epoch) : 0.0;
    __syncthreads();
    mark(s.mark, 0);
    if (par_off >= 0) {
        const uint64_t* yp = yfin + 2 * par_off;
        for (int i = threadIdx.x; i < kp; i += kThreads) s.rhs[i] = ll_load(yp + 2 * i, epoch);
    }
    if (e_smem) {
        mbar_wait(s.bar, par);
        par ^= 1u;
    }
    __syncthreads();
    mark(s.mark, 4);
    if (par_off >= 0 && k > 0) {
        if (e_smem)
            small_cols_dot(Es, kp, k, s.rhs, s.vb, s.red);  // E^T staged: out[r] = sum_c Es[c*k + r] v[c]
        else
            small_rows_dot(r_E + e_off, kp, k, kp, s.rhs, s.vb);
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += kThreads) s.va[i] += s.vb[i];
        __syncthreads();
    }
    mark(s.mark, 1);
    if (!leaf) {
        uint64_t* dst = yfin + 2 * yoff;
        for (int i = threadIdx.x; i < k; i += kThreads) ll_store(dst + 2 * i, s.va[i], epoch);
        mark(s.mark, 2);
        return;
    }
    const int size = (int)d[8];
    const int nv = (size * k + 1) & ~1;
    const bool v_smem = k > 0 && nv <= s.stage_bytes / 8;
    const double* Vg = r_V + v_off;
    if (v_smem) {  // (the E_t^T product above ended with a block barrier: Es is free)
        if (threadIdx.x == 0) {
            mbar_expect_tx(s.bar, 8u * (uint32_t)nv);
            bulk_g2s(Es, s.dpack + d[13] + ne, 8u * (uint32_t)nv, s.bar);
        }
        mbar_wait(s.bar, par);
    }
    __syncthreads();
    if (k > 0) {
        if (v_smem)
            small_cols_dot(Es, k, size, s.va, s.vb, nullptr);  // V^T staged
        else
            small_rows_dot(Vg, k, size, k, s.va, s.vb);
    }
    __syncthreads();
    const uint64_t* yn = ynear + 2 * (int64_t)start;
    for (int i = threadIdx.x; i < size; i += blockDim.x)
        y[row_perm[start + i]] = (sym ? s.yn[i] : ll_load(yn + 2 * i, epoch)) + (k > 0 ? s.vb[i] : 0.0);
}

// The band record is already in s.rec (kind in word 7: 0 near, 1 coupling).
template <bool kCoupling>
__device__ void task_band(const h2b_layout& L, const double* __restrict__ x, const uint64_t* xhat, uint64_t* out,
                          uint64_t* yfin, const uint64_t* ycpl, const uint64_t* ynear, double* y, uint32_t epoch,
                          const Shared& s) {
    const int64_t src_off = s.rec[0], gi_off = s.rec[3], out_off = s.rec[4];
    const int cols = (int)s.rec[1], rows = (int)s.rec[2];
    if (rows > 0 && cols > kChunkCols) {
        // wide row (a cluster with many couplings): the right-hand side is
        // gathered kChunkCols columns at a time so shared memory stays small;
        // rows <= kWarps (the host cuts such bands so), one row per warp, and
        // every lane walks its columns in the order rows_dot uses, carrying
        // its four chains across chunks (chunks are multiples of 128
        // columns): the same bits as the unchunked product
        const double* base = kCoupling ? L.S : L.D;
        const int64_t bytes = (int64_t)rows * cols * 8;
        const double* M = stage_issue(s, base + src_off, bytes);
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const double* row = M + (int64_t)min(warp, rows - 1) * cols;
        const int32_t* gidx = (kCoupling ? L.s_gidx : L.d_gidx) + gi_off;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = lane;
        for (int c0 = 0; c0 < cols; c0 += kChunkCols) {
            const int cn = min(kChunkCols, cols - c0);
            if (c0 > 0) __syncthreads();  // the previous chunk is consumed
            if (kCoupling)
                gather_ll(s.rhs, xhat, gidx + c0, cn, epoch);
            else
                gather(s.rhs, x, gidx + c0, cn);
            if (c0 == 0) mbar_wait(s.bar, s.parity);
            __syncthreads();
            const double* v = s.rhs - c0;
            if (warp < rows) {
                for (; c + 96 < cols && c < c0 + cn; c += 128) {
                    a0 = fma(row[c], v[c], a0);
                    a1 = fma(row[c + 32], v[c + 32], a1);
                    a2 = fma(row[c + 64], v[c + 64], a2);
                    a3 = fma(row[c + 96], v[c + 96], a3);
                }
                if (c0 + cn == cols)
                    for (; c < cols; c += 32) a0 = fma(row[c], v[c], a0);
            }
        }
        if (warp < rows) {
            double sum = (a0 + a1) + (a2 + a3);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) s.va[warp] = sum;
        }
        __syncthreads();
        uint64_t* dst = out + 2 * out_off;
        for (int i = threadIdx.x; i < rows; i += blockDim.x) ll_store(dst + 2 * i, s.va[i], epoch);
    } else if (rows > 0) {
        const double* base = kCoupling ? L.S : L.D;
        const int64_t bytes = (int64_t)rows * cols * 8;
        const double* M = stage_issue(s, base + src_off, bytes);
        mark(s.mark, 0);
        if (kCoupling)
            gather_ll(s.rhs, xhat, L.s_gidx + gi_off, cols, epoch);
        else
            gather(s.rhs, x, L.d_gidx + gi_off, cols);
        mark(s.mark, 1);
        if (kCoupling && s.pf >= 0) {
            // leaf final: its nearfield partial vectors (|t| LL words each) into L2 for near_sum
            const char* q = reinterpret_cast<const char*>(s.ppart + 2 * s.pf);
            const int lines = ((int)s.rec[16] * 16 + 127) / 128 + 1;
            for (int l = 0; l < lines; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(q + 128 * l));
        }
        mbar_wait(s.bar, s.parity);
        __syncthreads();
        mark(s.mark, 2);
        rows_dot(M, cols, rows, cols, s.rhs, s.va);
        __syncthreads();
        mark(s.mark, 3);
        uint64_t* dst = out + 2 * out_off;
        for (int i = threadIdx.x; i < rows; i += blockDim.x) ll_store(dst + 2 * i, s.va[i], epoch);
    }
    if (kCoupling && s.rec[5]) {
        __syncthreads();
        descent(L.r_E, L.r_V, L.row_perm, s.rec + 8, ycpl, yfin, ynear, y, epoch, s.rec[6] != 0, s,
                s.parity ^ (rows > 0 ? 1u : 0u));
    }
}

// Both products of a tall panel M (rows x cols, cols <= 64, row-major in
// shared memory) in ONE pass: lane l owns columns l and l + 32, warps take 8
// rows at a time.  Direct: y[r] = M[r,:] . xc (8 rows reduced together by
// recursive halving, stored by the lane that holds the row); transposed:
// z[c] = sum_r M[r,c] xr[r] (per-warp register sums, added in warp order).
// Fixed summation order throughout.
__device__ void panel_dot(const double* M, int rows, int cols, const double* xc, const double* xr, bool transposed,
                          uint64_t* yd, uint64_t* zt, int skip, double* red, uint32_t epoch) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool ok0 = lane < cols, ok1 = lane + 32 < cols;
    const double x0 = ok0 ? xc[lane] : 0.0, x1 = ok1 ? xc[lane + 32] : 0.0;
    double t0 = 0.0, t1 = 0.0;
#ifndef H2B_PANEL_R
#define H2B_PANEL_R 8
#endif
    constexpr int R = H2B_PANEL_R;
    constexpr int lg = log2c(R);
    int ri = 0;
#pragma unroll
    for (int j = 0; j < lg; ++j) ri |= ((lane >> (4 - j)) & 1) << (lg - 1 - j);
    for (int rb = R * warp; rb < rows; rb += R * kWarps) {
        double a[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int r = rb + k;
            double m0 = 0.0, m1 = 0.0, xv = 0.0;
            if (r < rows) {
                if (ok0) m0 = M[r * cols + lane];
                if (ok1) m1 = M[r * cols + lane + 32];
                xv = xr[r];
            }
            a[k] = fma(m1, x1, m0 * x0);
            t0 = fma(m0, xv, t0);
            t1 = fma(m1, xv, t1);
        }
        const double sum = warp_sum<R>(a, lane);
        if ((lane & ((32 / R) - 1)) == 0 && rb + ri < rows) ll_store(yd + 2 * (rb + ri), sum, epoch);
    }
    if (!transposed) return;
    red[warp * 64 + lane] = t0;
    red[warp * 64 + 32 + lane] = t1;
    __syncthreads();
    for (int c = skip + threadIdx.x; c < cols; c += kThreads) {
        double z = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) z += red[w * 64 + c];
        ll_store(zt + 2 * c, z, epoch);
    }
}

// Gather two index lists in one pass (all index loads, then all value loads):
// d1[i] = src[idx1[i]], i < n1, and d2[i] = src[idx2[i]], i < n2.
__device__ __forceinline__ void gather2(double* d1, const int32_t* idx1, int n1, double* d2, const int32_t* idx2,
                                        int n2, const double* __restrict__ src) {
    constexpr int kU = 4;
    const int n = n1 + n2;
    for (int base = 0; base < n; base += kU * kThreads) {
        int ix[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = base + u * kThreads + (int)threadIdx.x;
            ix[u] = i < n1 ? __ldg(idx1 + i) : i < n ? __ldg(idx2 + (i - n1)) : -1;
        }
        double v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = ix[u] >= 0 ? __ldg(src + ix[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = base + u * kThreads + (int)threadIdx.x;
            if (i < n1)
                d1[i] = v[u];
            else if (i < n)
                d2[i - n1] = v[u];
        }
    }
}

// Symmetric nearfield band: one column panel [D_(t,s) ...] (all rows of row
// leaf t, upper blocks s >= t in leaf order, the diagonal block first) streamed
// ONCE for both triangles: the direct product D x|_cols -> t's partial at
// out_off, and the transposed product D^T x|_t -> the columns' partials at
// tr_off + c (skipped for the diagonal block's columns, which are stored in
// full).  Never waits.
__device__ void task_panel(const double* __restrict__ base, const int32_t* __restrict__ gl,
                           const double* __restrict__ x, uint64_t* ppart, uint32_t epoch, const Shared& s) {
    const int64_t src_off = s.rec[0], gi_off = s.rec[3], out_off = s.rec[4];
    const int cols = (int)s.rec[1], rows = (int)s.rec[2];
    const int64_t tr_off = s.rec[8], rg_off = s.rec[10];
    const int skip = (int)s.rec[9];
    const int64_t bytes = ((int64_t)rows * cols * 8 + 15) & ~int64_t(15);  // panels are padded to 16 bytes
    const double* M = stage_issue(s, base + src_off, bytes);
    mark(s.mark, 0);
    const bool tr = skip < cols;
    gather2(s.rhs, gl + gi_off, cols, s.vb, gl + rg_off, tr ? rows : 0, x);
    mark(s.mark, 1);
    mbar_wait(s.bar, s.parity);
    __syncthreads();
    mark(s.mark, 2);
    panel_dot(M, rows, cols, s.rhs, s.vb, tr, ppart + 2 * out_off, ppart + 2 * tr_off, skip, s.red, epoch);
    mark(s.mark, 3);
}

struct KArgs {
    h2b_layout L;
    const int64_t* rec;
    const int64_t* fwd_off;
    int64_t band_base, band_bytes, dgidx_bytes;
    int n_near, n_cpl, n_near_a, n_inner_bands;
    int n_fwd;         // forward tasks of this launch (tickets [0, n_fwd))
    int max_cols, vec_len, stage_bytes;
    int64_t e_bytes_r;
    uint64_t *xhat, *ycpl, *yfin, *ynear;
    unsigned long long* ctrl;
    unsigned long long* trace;
    const double* dsym;      // symmetric nearfield (null: not used)
    const int32_t* gsym;
    uint64_t* ppart;
    const int64_t* nsum;
    const double* dpack;     // downward-step operands (transposed row basis)
};

#ifndef H2B_MINB
#define H2B_MINB 6
#endif

// One task (tickets [0, c_leaves): forward; then band / descent records).
template <bool kTrace>
__device__ __forceinline__ void run_task(const KArgs& a, const double* __restrict__ x, double* __restrict__ y,
                                         const int ticket, const uint32_t epoch, Shared& s) {
    const h2b_layout& L = a.L;
    unsigned long long t_begin = 0;
    if (kTrace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    s.mark = kTrace ? a.trace + 8 * ticket + 3 : nullptr;
    const int tB = a.n_fwd;

    if (ticket < tB) {
        // pull the band records, the nearfield gather lists and x into L2 for
        // the streaming tasks that follow (fire-and-forget; LL needs no fences)
        // (records and lists only when they fit L2 beside everything else:
        // launch_matvec passes zero lengths otherwise)
        prefetch_slice(reinterpret_cast<const double*>(a.rec + a.band_base), a.band_bytes, ticket, a.n_fwd);
        prefetch_slice(reinterpret_cast<const double*>(a.dsym ? a.gsym : L.d_gidx), a.dgidx_bytes, ticket,
                       a.n_fwd);
        prefetch_slice(x, 8 * L.n_cols, ticket, a.n_fwd);
        // the record of the forward task kFwdAhead tickets on (no dependent load)
        if (threadIdx.x == 64 && ticket + kFwdAhead < a.n_fwd)
            bulk_prefetch_l2(a.rec + (int64_t)kFwdStride * (ticket + kFwdAhead), 8 * kFwdStride);
        task_forward(L.c_V, L.c_E, L.col_perm, a.rec + (int64_t)kFwdStride * ticket, x, a.xhat, epoch, s, a.rec);
    } else {
        const int b = ticket - tB;
        load_rec(s, a.rec + a.band_base + (int64_t)kBandWords * b, kBandWords);
        const int kind = (int)s.rec[7];
        // a cluster's last band: pull its downward-step operands into L2 now
        // (the bulk copy after the band's product then hits L2)
        if (kind == kKindCpl && s.rec[5] && s.rec[22] > 0 && threadIdx.x == 32)
            bulk_prefetch_l2(a.dpack + s.rec[21], (uint32_t)s.rec[22]);
        // ... and a leaf's nearfield partial vectors (symmetric nearfield; summed by
        // near_sum after the band's product): list entry m -> the |t| LL words at
        // ppart + 2 list[m], one 128-byte line per 8 rows
        // (the list entry is loaded here and used after the band's gather is under way, task_band)
        s.pf = -1;
        if (kind == kKindCpl && s.rec[5] && a.ppart && s.rec[13] && (int)threadIdx.x < (int)s.rec[20])
            s.pf = __ldg(a.nsum + s.rec[19] + threadIdx.x);
        if (kind == kKindNearSym)
            task_panel(a.dsym, a.gsym, x, a.ppart, epoch, s);
        else if (kind == kKindNear)
            task_band<false>(L, x, a.xhat, a.ynear, a.yfin, a.ycpl, a.ynear, y, epoch, s);
        else
            task_band<true>(L, x, a.xhat, a.ycpl, a.yfin, a.ycpl, a.ynear, y, epoch, s);
    }
    if (kTrace) {
        // (diagnostic instantiation only: the product kernel ends with its task)
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t_end;
            unsigned smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            a.trace[8 * ticket] = t_begin;
            a.trace[8 * ticket + 1] = t_end;
            const int kd = ticket < tB ? 2 : (int)s.rec[7];
            a.trace[8 * ticket + 2] = smid | ((unsigned long long)kd << 16) |
                                      (kd == 2 ? (unsigned long long)s.rec[5] << 24 : 0ull) |
                                      (kd == 1 && s.rec[5] ? (1ull << 41) | ((unsigned long long)s.rec[17] << 32) : 0ull);
        }
    }
}



template <bool kTrace>
__global__ void __launch_bounds__(kThreads, H2B_MINB) k_matvec(const KArgs a, const double* __restrict__ x,
                                                       double* __restrict__ y) {
    extern __shared__ __align__(128) char smraw[];
    __shared__ int s_ticket;
    __shared__ uint32_t s_epoch;
    __shared__ int64_t s_rec[kFwdHead + kFwdLevel * kMaxDepth];
    Shared s;
    s.bar = reinterpret_cast<uint64_t*>(smraw);
    s.stage = smraw + 128;
    s.stage_bytes = a.stage_bytes;
    s.rhs = reinterpret_cast<double*>(smraw + 128 + a.stage_bytes);
    s.va = s.rhs + a.max_cols;
    s.vb = s.va + 2 * a.vec_len;
    s.red = s.vb + a.vec_len;
    s.yn = s.red + kWarps * 64;
    s.near_sym = a.dsym != nullptr;
    s.ppart = a.ppart;
    s.nsum = a.nsum;
    s.dpack = a.dpack;
    s.rec = s_rec;
    s.parity = 0;
    if (threadIdx.x == 0) {
        // tickets count on across launches: launch = t / grid (every CTA of a
        // launch takes exactly one ticket before the next launch starts)
        // (odd epochs: the x_hat-exchange entry points compute theirs on the host)
        const unsigned long long t = atomicAdd(a.ctrl, 1ull);
        s_ticket = (int)(t % gridDim.x);
        s_epoch = 2u * (uint32_t)(t / gridDim.x) + 1u;
        mbar_init(s.bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ticket = s_ticket;
    const uint32_t epoch = s_epoch;
    run_task<kTrace>(a, x, y, ticket, epoch, s);
}

// ---- x_hat exchange (row-sharded plans, SURVEY 8(e) "better variant") ------
// pack: this rank's coefficients (LL, forward launch) -> plain send buffer;
// one warp per cluster
__global__ void k_xhat_pack(h2b_layout L, const uint64_t* __restrict__ xhat_f, uint32_t epoch,
                            const int32_t* __restrict__ own, const int64_t* __restrict__ own_off, int n,
                            double* __restrict__ send) {
    const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (w >= n) return;
    const int u = own[w];
    const int k = L.c_rank[u];
    const int64_t xo = L.c_xhat_off[u], so = own_off[w];
    for (int c = lane; c < k; c += 32) send[so + c] = ll_load(xhat_f + 2 * (xo + c), epoch);
}

// import: gathered coefficients -> LL x_hat of the next bands launch (and a
// plain copy for the spanning climbs)
__global__ void k_xhat_import(h2b_layout L, const double* __restrict__ recv, const int32_t* __restrict__ imp,
                              const int64_t* __restrict__ src, int n, uint64_t* __restrict__ xhat, uint32_t epoch,
                              double* __restrict__ plain) {
    const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (w >= n) return;
    const int u = imp[w];
    const int k = L.c_rank[u];
    const int64_t xo = L.c_xhat_off[u], so = src[w];
    for (int c = lane; c < k; c += 32) {
        const double v = recv[so + c];
        plain[xo + c] = v;
        ll_store(xhat + 2 * (xo + c), v, epoch);
    }
}

// a cluster spanning several ranks: x_hat_p = E_c0^T x_hat_c0 + E_c1^T x_hat_c1
// with exactly the arithmetic of the forward climb in task_forward /
// forward_warp (same branch on rank and staging size), so the coefficients
// are the bits one GPU computes.  One 128-thread CTA per cluster.
__global__ void __launch_bounds__(kThreads) k_xhat_climb(h2b_layout L, const int32_t* __restrict__ nodes, int stage_bytes,
                                                       int vec_len, double* __restrict__ plain,
                                                       uint64_t* __restrict__ xhat, uint32_t epoch) {
    extern __shared__ __align__(16) double sm[];
    double* buf = sm;                                  // stage_bytes: [E_c0; E_c1]
    double* va = sm + stage_bytes / 8;                 // 2 vec_len
    double* vb = va + 2 * vec_len;                     // vec_len
    double* rhs = vb + vec_len;                        // vec_len
    double* red = rhs + vec_len;                       // kWarps * 64
    const int p = nodes[blockIdx.x];
    const int c0 = L.c_child[2 * p], c1 = L.c_child[2 * p + 1];
    const int k0 = L.c_rank[c0], k1 = L.c_rank[c1], kp = L.c_rank[p];
    const int n0 = k0 * kp, n1 = k1 * kp;
    const bool in_smem = (n0 + n1) * 8 <= stage_bytes;
    const double* E0 = L.c_E + L.c_e_off[c0];
    const double* E1 = L.c_E + L.c_e_off[c1];
    if (in_smem) {
        for (int i = threadIdx.x; i < n0; i += kThreads) buf[i] = E0[i];
        for (int i = threadIdx.x; i < n1; i += kThreads) buf[n0 + i] = E1[i];
    }
    for (int r = threadIdx.x; r < k0; r += kThreads) va[r] = plain[L.c_xhat_off[c0] + r];
    for (int r = threadIdx.x; r < k1; r += kThreads) va[k0 + r] = plain[L.c_xhat_off[c1] + r];
    __syncthreads();
    if (in_smem && kp <= 32) {
        if (threadIdx.x < kp) vb[threadIdx.x] = climb_coef(buf, buf + n0, k0, k1, kp, va, threadIdx.x);
        __syncthreads();
    } else if (in_smem) {
        small_cols_dot(buf, k0 + k1, kp, va, vb, red);
        __syncthreads();
    } else {
        cols_dot(E0, k0, kp, va, red, vb);
        for (int c = threadIdx.x; c < kp; c += kThreads) rhs[c] = vb[c];
        __syncthreads();
        cols_dot(E1, k1, kp, va + k0, red, vb);
        for (int c = threadIdx.x; c < kp; c += kThreads) vb[c] += rhs[c];
        __syncthreads();
    }
    const int64_t xo = L.c_xhat_off[p];
    for (int c = threadIdx.x; c < kp; c += kThreads) {
        plain[xo + c] = vb[c];
        ll_store(xhat + 2 * (xo + c), vb[c], epoch);
    }
}

// Plan creation: the operands of every downward step, transposed into the
// layout the step's products read (one CTA per step): E_t^T (k_parent x k),
// then V_t^T (k x |t|) for leaves; see descent().
__global__ void k_pack_descent(const double* __restrict__ r_E, const double* __restrict__ r_V,
                               const int64_t* __restrict__ desc, double* __restrict__ pack) {
    const int64_t* d = desc + 6 * (int64_t)blockIdx.x;
    const int64_t e_off = d[0], v_off = d[3];
    const int k = (int)d[1], kp = (int)d[2], size = (int)d[4];
    double* out = pack + d[5];
    if (e_off >= 0)
        for (int i = threadIdx.x; i < k * kp; i += blockDim.x) {
            const int r = i / kp, c = i - r * kp;
            out[(int64_t)c * k + r] = r_E[e_off + i];
        }
    out += (((int64_t)k * kp + 1) & ~int64_t(1));
    if (v_off >= 0)
        for (int i = threadIdx.x; i < size * k; i += blockDim.x) {
            const int r = i / k, c = i - r * k;
            out[(int64_t)c * size + r] = r_V[v_off + i];
        }
}

__global__ void k_diagonal(h2b_layout L, double* __restrict__ diag) {
    // row-sharded plans: only the rank's own leaves (row_perm maps its rows)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (L.owned ? L.n_owned : L.r_nodes)) return;
    const int node = L.owned ? L.owned[i] : i;
    if (L.r_v_off[node] < 0) return;
    if (L.owned && (L.r_start[node] + L.r_size[node] > L.n_rows || L.row_perm[L.r_start[node]] < 0)) return;
    const int ts = L.r_start[node], te = ts + L.r_size[node];
    const int C = L.d_cols[node];
    const double* D = L.D + L.d_off[node];
    for (int r = ts; r < te; ++r) {
        double acc = 0.0;
        int off = 0;
        for (int f = L.near_ptr[node]; f < L.near_ptr[node + 1]; ++f) {
            const int s = L.near_col[f];
            const int ss = L.c_start[s], sz = L.c_size[s];
            if (r >= ss && r < ss + sz) acc += D[(int64_t)(r - ts) * C + off + (r - ss)];
            off += sz;
        }
        diag[L.row_perm[r]] = acc;
    }
}

template <typename T>
cudaError_t fetch(const T* d, int64_t n, std::vector<T>& h) {
    h.resize((size_t)std::max<int64_t>(n, 0));
    return n > 0 ? cudaMemcpy(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost) : cudaSuccess;
}

}  // namespace
}  // namespace h2b

using namespace h2b;

namespace h2b {
namespace {

// D(t,s)[a][b] == D(s,t)[b][a] bit for bit, per upper block pair (job words:
// off1, ld1, off2, ld2, rows, cols); any mismatch sets *bad.
__global__ void k_sym_check(const double* __restrict__ D, const int64_t* __restrict__ jobs,
                            int* __restrict__ bad) {
    const int64_t* j = jobs + 6 * (int64_t)blockIdx.x;
    const int64_t o1 = j[0], l1 = j[1], o2 = j[2], l2 = j[3];
    const int nr = (int)j[4], nc = (int)j[5];
    int mism = 0;
    for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
        const int a = e / nc, b = e - a * nc;
        mism |= __double_as_longlong(D[o1 + a * l1 + b]) != __double_as_longlong(D[o2 + b * l2 + a]);
    }
    if (__syncthreads_or(mism) && threadIdx.x == 0) atomicOr(bad, 1);
}

// Column panels of the symmetric nearfield (job words: source row base,
// source ld, rows, cols, destination, source-column list offset).
__global__ void k_sym_pack(const double* __restrict__ D, const int64_t* __restrict__ jobs,
                           const int32_t* __restrict__ srccol, double* __restrict__ out) {
    const int64_t* j = jobs + 6 * (int64_t)blockIdx.x;
    const int64_t src = j[0], ld = j[1], dst = j[4], so = j[5];
    const int nr = (int)j[2], nc = (int)j[3];
    for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
        const int a = e / nc, b = e - a * nc;
        out[dst + e] = D[src + a * ld + __ldg(srccol + so + b)];
    }
}

// Host side of the symmetric nearfield (plans whose row and column trees
// coincide and whose nearfield is symmetric bit for bit, e.g. the
// single-layer Galerkin matrix, containers.py near_slp_jobs).  Per row leaf t,
// the blocks it streams are cut into column panels of all |t| rows that fit
// the TMA stage, in the column order
//   [ diagonal block | one-sided blocks | upper paired blocks ]
// where "paired" blocks (t, s) have their mirror (s, t) held by the same plan
// and start(s) > start(t): their transposed product is s's contribution from
// this panel.  The first `skip` columns have no transposed output.  Single-GPU
// plans pair every block; a row-sharded plan (L.owned) holds only its own
// leaves' blocks, so blocks towards another rank's leaves are one-sided.
struct SymNear {
    bool on = false;
    std::vector<std::vector<int64_t>> bands;  // per row node: band records
    std::vector<int64_t> list_off, list_n;    // per row node: its partial list
    std::vector<int64_t> nsum, pack, check;
    std::vector<int32_t> srccol, gsym;
    std::vector<std::vector<int>> producers;  // per leaf u: the leaves t whose panels hold (t, u)
    int64_t dsym_len = 0, ppart_len = 0, near_bytes = 0;
};

// Staging buffer of a plan: the TMA stage plus the rest of the CTA's shared
// memory (other_smem: the gathered right-hand side and vectors) decide how
// many CTAs an SM holds (at most H2B_MINB by registers).  Measured (sphere
// L6 / L8 / L9-m5, 16-40 KB): 24 KB at 6 CTAs/SM is best where it fits
// (L6 56 us vs 62 us at 28 KB; L8 765 vs 838 us); where the wide coupling rows
// of config 3 leave room for only 5 CTAs at 24 KB, 20 KB at 6 CTAs wins
// (3.63 vs 3.81 ms).  So: the largest stage <= 24 KB that keeps H2B_MINB CTAs
// per SM, else the one with the most bytes in flight per SM.  H2B_STAGE_KB
// overrides (tuning experiments).
int plan_stage_bytes(int other_smem) {
    if (const char* e = getenv("H2B_STAGE_KB")) {
        const int kb = atoi(e);
        if (kb * 1024 >= kStageMin && kb * 1024 <= kStageMax) return kb * 1024;
    }
    constexpr int kSmPerSM = 233472, kPerCtaFixed = 1024 + 1792;  // driver reserve + static shared memory
    auto ctas = [&](int st) { return std::min(H2B_MINB, kSmPerSM / (st + other_smem + kPerCtaFixed)); };
    for (int st = 24 * 1024; st >= kStageMin; st -= 4096)
        if (ctas(st) >= H2B_MINB) return st;
    int best = kStageMin;
    int64_t best_score = -1;
    for (int st = kStageMin; st <= kStageMax; st += 4096) {
        const int64_t score = (int64_t)ctas(st) * st;
        if (ctas(st) >= 1 && score >= best_score) {
            best_score = score;
            best = st;
        }
    }
    return best;
}

int build_sym_near(int stage_bytes, const h2b_layout& L, const std::vector<int32_t>& rstart, const std::vector<int32_t>& rsize,
                   const std::vector<int32_t>& cstart, const std::vector<int32_t>& csize,
                   const std::vector<int64_t>& rvoff, const std::vector<int32_t>& dcols,
                   const std::vector<int64_t>& doff, const std::vector<int64_t>& dgoff, SymNear& S) {
    S.on = false;
    if (L.r_nodes != L.c_nodes || L.n_rows != L.n_cols || !L.near_ptr || !L.near_col) return 0;
    if (const char* e = getenv("H2B_NEAR_SYM"))
        if (e[0] == '0') return 0;
    const int n = L.r_nodes;
    for (int u = 0; u < n; ++u)
        if (rstart[u] != cstart[u] || rsize[u] != csize[u]) return 0;
    if (!L.owned) {
        // (row-sharded plans map rows and columns to different index spaces;
        // there the trees are checked by the structure above)
        std::vector<int64_t> rp, cp;
        H2B_CUDA_TRY(fetch(L.row_perm, L.n_rows, rp));
        H2B_CUDA_TRY(fetch(L.col_perm, L.n_cols, cp));
        if (rp != cp) return 0;
    }
    std::vector<int32_t> nptr, ncol, dg;
    H2B_CUDA_TRY(fetch(L.near_ptr, (int64_t)n + 1, nptr));
    H2B_CUDA_TRY(fetch(L.near_col, std::max<int64_t>(nptr[n], 1), ncol));
    int64_t glen = 0;
    for (int u = 0; u < n; ++u)
        if (rvoff[u] >= 0) glen = std::max<int64_t>(glen, dgoff[u] + dcols[u]);
    H2B_CUDA_TRY(fetch(L.d_gidx, std::max<int64_t>(glen, 1), dg));
    // leaves whose tasks this plan runs (all leaves on one GPU; a rank's own)
    std::vector<char> mine(n, 1);
    if (L.owned) {
        std::vector<int32_t> own;
        H2B_CUDA_TRY(fetch(L.owned, L.n_owned, own));
        std::fill(mine.begin(), mine.end(), 0);
        for (int u : own)
            if (u >= 0 && u < n) mine[u] = 1;
    }
    std::vector<char> has(n, 0);
    std::vector<std::vector<std::pair<int, int64_t>>> blocks(n);  // (s, column offset in t's row)
    for (int t = 0; t < n; ++t) {
        int64_t c = 0;
        for (int q = nptr[t]; q < nptr[t + 1]; ++q) {
            const int s = ncol[q];
            if (rvoff[t] < 0 || s < 0 || s >= n || rvoff[s] < 0) return 0;
            blocks[t].push_back({s, c});
            c += rsize[s];
        }
        has[t] = mine[t] && nptr[t + 1] > nptr[t];
    }
    auto find = [&](int t, int s) -> int64_t {
        for (const auto& b : blocks[t])
            if (b.first == s) return b.second;
        return -1;
    };
    for (int t = 0; t < n; ++t) {
        if (rvoff[t] < 0) continue;
        if (!has[t]) {
            if (!L.owned) return 0;  // one GPU: every leaf has its diagonal block
            continue;
        }
        if (find(t, t) < 0) return 0;
        for (const auto& b : blocks[t])
            if (has[b.first] && find(b.first, t) < 0) return 0;  // a held leaf must hold the mirror
            else if (!has[b.first] && !L.owned) return 0;
    }
    // per leaf: diagonal, one-sided, then upper paired blocks; check jobs for
    // the bitwise symmetry test of the paired (and diagonal) blocks
    std::vector<std::vector<std::pair<int, int64_t>>> up(n);
    std::vector<int64_t> skip_w(n, 0);  // columns without a transposed output
    for (int t = 0; t < n; ++t) {
        if (rvoff[t] < 0 || !has[t]) continue;
        up[t].push_back({t, find(t, t)});
        skip_w[t] = rsize[t];
        for (const auto& b : blocks[t])
            if (b.first != t && !has[b.first]) {
                up[t].push_back(b);
                skip_w[t] += rsize[b.first];
            }
        for (const auto& b : blocks[t])
            if (b.first != t && has[b.first] && rstart[b.first] > rstart[t]) up[t].push_back(b);
        for (const auto& b : up[t])
            if (has[b.first])
                S.check.insert(S.check.end(), {doff[t] + b.second, dcols[t], doff[b.first] + find(b.first, t),
                                               dcols[b.first], rsize[t], rsize[b.first]});
    }
    // panels, partial offsets
    S.bands.assign(n, {});
    S.list_off.assign(n, 0);
    S.list_n.assign(n, 0);
    S.producers.assign(n, {});
    std::vector<int64_t> tbase(n, 0);
    std::vector<std::vector<int64_t>> tcol(n);  // per t: column offset of each streamed block in its panels
    std::vector<std::vector<int64_t>> direct(n);
    int64_t pdir = 0, dlen = 0, g = 0;
    for (int t = 0; t < n; ++t) {
        if (rvoff[t] < 0 || !has[t]) continue;
        const int rows = rsize[t];
        int64_t W = 0;
        for (const auto& b : up[t]) {
            tcol[t].push_back(W);
            W += rsize[b.first];
        }
        int wmax = std::min(64, std::max(2, (int)(stage_bytes / 8 / std::max(rows, 1))));
        if ((rows & 1) && (wmax & 1)) --wmax;
        const int64_t gbase = g;
        for (const auto& b : up[t])
            for (int j = 0; j < rsize[b.first]; ++j) {
                S.srccol.push_back((int32_t)(b.second + j));
                S.gsym.push_back(dg[dgoff[t] + b.second + j]);
            }
        g += W;
        for (int64_t j0 = 0; j0 < W; j0 += wmax) {
            const int w = (int)std::min<int64_t>(wmax, W - j0);
            const int skip = (int)std::max<int64_t>(0, std::min<int64_t>(w, skip_w[t] - j0));
            std::vector<int64_t> r(kBandWords, 0);
            r[0] = dlen;
            r[1] = w;
            r[2] = rows;
            r[3] = gbase + j0;
            r[4] = pdir;
            r[7] = kKindNearSym;
            r[8] = j0;  // + tbase[t] below
            r[9] = skip;
            r[10] = gbase;  // t's own x: the diagonal block's columns come first
            S.bands[t].insert(S.bands[t].end(), r.begin(), r.end());
            S.pack.insert(S.pack.end(), {doff[t], dcols[t], rows, w, dlen, gbase + j0});
            direct[t].push_back(pdir);
            pdir += rows;
            dlen += ((int64_t)rows * w + 1) & ~int64_t(1);  // 16-byte aligned panels
            S.near_bytes += 8 * (int64_t)rows * w;
        }
        tbase[t] = W;  // temporarily: the width
    }
    int64_t tpos = pdir;
    for (int t = 0; t < n; ++t) {
        if (rvoff[t] < 0 || !has[t]) continue;
        const int64_t W = tbase[t];
        tbase[t] = tpos;
        tpos += W;
        for (size_t i = 0; i < S.bands[t].size(); i += kBandWords) S.bands[t][i + 8] += tpos - W;
    }
    S.ppart_len = tpos;
    S.dsym_len = dlen;
    // per leaf u: its panels' direct partials, then the transposed partials
    // of the paired blocks (t, u) with t before u, in u's near-list order
    for (int u = 0; u < n; ++u) {
        if (rvoff[u] < 0 || !has[u]) continue;
        S.list_off[u] = (int64_t)S.nsum.size();
        for (int64_t o : direct[u]) S.nsum.push_back(o);
        for (const auto& b : blocks[u]) {
            const int t = b.first;
            if (t == u || !has[t] || rstart[t] > rstart[u]) continue;
            int64_t off = -1;
            for (size_t i = 0; i < up[t].size(); ++i)
                if (up[t][i].first == u) off = tbase[t] + tcol[t][i];
            if (off < 0) return 0;
            S.nsum.push_back(off);
            S.producers[u].push_back(t);
        }
        S.list_n[u] = (int64_t)S.nsum.size() - S.list_off[u];
    }
    S.on = true;
    return 0;
}

}  // namespace
}  // namespace h2b

namespace {
constexpr int kSymNear = 1;
int plan_create(const h2b_layout* layout, h2b_plan** out, int sym_flags, const int8_t* cmask = nullptr) {
    if (!layout || !out) return fail(H2B_ERR_INVALID, "h2b_plan_create: null pointer");
    const h2b_layout& L = *layout;
    if (L.c_nodes <= 0 || L.r_nodes <= 0 || L.c_leaves <= 0) return fail(H2B_ERR_INVALID, "h2b_plan_create: empty tree");
    if (!L.d_gidx || !L.d_goff || !L.s_gidx || !L.s_goff)
        return fail(H2B_ERR_INVALID, "h2b_plan_create: gather indices missing");
    // host copies of the layout (plan creation only)
    std::vector<int32_t> scols, dcols, rsize, rstart, rrank, rparent, crank, csize, cstart, cparent, cchild, order,
        leaves;
    std::vector<int64_t> rvoff, reoff, ryoff, soff, doff, sgoff, dgoff, cvoff, ceoff, cxoff;
    H2B_CUDA_TRY(fetch(L.s_cols, L.r_nodes, scols));
    H2B_CUDA_TRY(fetch(L.d_cols, L.r_nodes, dcols));
    H2B_CUDA_TRY(fetch(L.r_size, L.r_nodes, rsize));
    H2B_CUDA_TRY(fetch(L.r_start, L.r_nodes, rstart));
    H2B_CUDA_TRY(fetch(L.r_rank, L.r_nodes, rrank));
    H2B_CUDA_TRY(fetch(L.r_parent, L.r_nodes, rparent));
    H2B_CUDA_TRY(fetch(L.c_rank, L.c_nodes, crank));
    H2B_CUDA_TRY(fetch(L.c_size, L.c_nodes, csize));
    H2B_CUDA_TRY(fetch(L.c_start, L.c_nodes, cstart));
    H2B_CUDA_TRY(fetch(L.c_parent, L.c_nodes, cparent));
    H2B_CUDA_TRY(fetch(L.c_child, 2 * (int64_t)L.c_nodes, cchild));
    H2B_CUDA_TRY(fetch(L.c_leaf_list, L.c_leaves, leaves));
    H2B_CUDA_TRY(fetch(L.r_v_off, L.r_nodes, rvoff));
    H2B_CUDA_TRY(fetch(L.r_e_off, L.r_nodes, reoff));
    H2B_CUDA_TRY(fetch(L.r_yhat_off, L.r_nodes, ryoff));
    H2B_CUDA_TRY(fetch(L.s_off, L.r_nodes, soff));
    H2B_CUDA_TRY(fetch(L.d_off, L.r_nodes, doff));
    H2B_CUDA_TRY(fetch(L.s_goff, L.r_nodes, sgoff));
    H2B_CUDA_TRY(fetch(L.d_goff, L.r_nodes, dgoff));
    H2B_CUDA_TRY(fetch(L.c_v_off, L.c_nodes, cvoff));
    H2B_CUDA_TRY(fetch(L.c_e_off, L.c_nodes, ceoff));
    H2B_CUDA_TRY(fetch(L.c_xhat_off, L.c_nodes, cxoff));
    if (L.owned) {
        H2B_CUDA_TRY(fetch(L.owned, L.n_owned, order));
    } else {
        H2B_CUDA_TRY(fetch(L.r_order, L.r_nodes, order));
    }
    int maxcols = 2, maxk = 0, maxleaf = 0;
    for (int i = 0; i < L.r_nodes; ++i) {
        maxcols = std::max(maxcols, std::max(scols[i], dcols[i]));
        maxk = std::max(maxk, rrank[i]);
        if (rvoff[i] >= 0) maxleaf = std::max(maxleaf, rsize[i]);
    }
    for (int i = 0; i < L.c_nodes; ++i) maxk = std::max(maxk, crank[i]);
    for (int l : leaves) maxleaf = std::max(maxleaf, csize[l]);
    maxcols = std::max(maxcols, maxk);
    if (maxk > kMaxVec || maxleaf > kMaxVec)
        return fail(H2B_ERR_INVALID, "h2b_plan_create: cluster rank or leaf size above 512");
    const int vec_len = (std::max(maxk, maxleaf) + 1) & ~1;
    // symmetric nearfield: each leaf's partials are summed in the leaf's final
    // task (separate sum tasks in the nearfield stream measured slower)
    // gathered right-hand side per task: a panel (<= 64 columns) where the
    // symmetric layouts are used, else the widest row of D / S
    auto cols_needed = [&](bool sym_on) {
        int mc = std::max(2, maxk);
        for (int i = 0; i < L.r_nodes; ++i) {
            mc = std::max(mc, sym_on ? std::min<int>(dcols[i], 64) : dcols[i]);
            mc = std::max(mc, scols[i]);
        }
        return std::min((mc + 1) & ~1, std::max(kChunkCols, (maxk + 1) & ~1));
    };
    auto other_smem = [&](bool sym_on) {
        return 128 + (int)sizeof(double) * (cols_needed(sym_on) + 3 * vec_len +
                                             (sym_on ? 2 * vec_len + kWarps * 64 : kWarps * 32));
    };
    // symmetric nearfield: each leaf's partials are summed in the leaf's final
    // task (separate sum tasks in the nearfield stream measured slower)
    const bool want_sym = (sym_flags & kSymNear) != 0;
    const int stage = plan_stage_bytes(other_smem(want_sym));
    SymNear sym;
    if (want_sym)
        if (int rc = build_sym_near(stage, L, rstart, rsize, cstart, csize, rvoff, dcols, doff, dgoff, sym)) return rc;
    maxcols = cols_needed(sym.on);
    const int smem = stage + other_smem(sym.on);
    if (smem > 227 * 1024) return fail(H2B_ERR_INVALID, "h2b_plan_create: gathered right-hand side exceeds shared memory");

    std::vector<int64_t> rec, fwd_off;
    // Skip the zero work at the top of the trees: x_hat_u is needed only if u
    // or an ancestor is the column cluster of a far block; v_t is non-zero only
    // if t or an ancestor has couplings (for the reference geometries the top
    // levels are all nearfield, e.g. depths 0-3 at config 1).  The forward climb
    // stops below the first needed level and the downward chain starts there.
    std::vector<char> need_c(L.c_nodes, 0), hasv(L.r_nodes, 0);
    {
        std::vector<int32_t> fptr, fcol;
        H2B_CUDA_TRY(fetch(L.far_ptr, (int64_t)L.r_nodes + 1, fptr));
        H2B_CUDA_TRY(fetch(L.far_col, std::max<int64_t>(fptr[L.r_nodes], 0), fcol));
        for (int32_t c : fcol) need_c[c] = 1;
        auto top_down = [](int n, const std::vector<int32_t>& parent, std::vector<char>& flag) {
            std::vector<int> depth(n, -1), idx(n);
            for (int u = 0; u < n; ++u) {
                int d = 0;
                for (int q = parent[u]; q >= 0; q = parent[q]) ++d;
                depth[u] = d;
                idx[u] = u;
            }
            std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return depth[a] < depth[b]; });
            for (int u : idx)
                if (parent[u] >= 0 && flag[parent[u]]) flag[u] = 1;
        };
        top_down(L.c_nodes, cparent, need_c);
        for (int u = 0; u < L.r_nodes; ++u) hasv[u] = (scols[u] > 0 && rrank[u] > 0) ? 1 : 0;
        top_down(L.r_nodes, rparent, hasv);
    }
    // A: forward records: fixed-stride headers (with the leaf's first 64 x
    // indices), then per task the levels it climbs as the right child
    std::vector<int> fleaves;
    for (int i = 0; i < L.c_leaves; ++i)
        if (!cmask || cmask[leaves[i]]) fleaves.push_back(leaves[i]);  // x_hat exchange: this rank's column leaves only
    std::vector<int64_t> cperm;
    H2B_CUDA_TRY(fetch(L.col_perm, L.n_cols, cperm));
    rec.assign((size_t)kFwdStride * fleaves.size(), 0);
    for (size_t fi = 0; fi < fleaves.size(); ++fi) {
        const int leaf = fleaves[fi];
        fwd_off.push_back((int64_t)(kFwdStride * fi));
        const size_t hdr = (size_t)kFwdStride * fi;
        {
            const int64_t h[kFwdHead] = {cstart[leaf], csize[leaf], crank[leaf], cvoff[leaf], cxoff[leaf], 0, 0,
                                         (int64_t)rec.size()};
            std::copy(h, h + kFwdHead, rec.begin() + hdr);
            int32_t ix[2 * (kFwdStride - kFwdHead)] = {0};
            for (int r = 0; r < std::min<int>(csize[leaf], 2 * (kFwdStride - kFwdHead)); ++r) {
                const int64_t q = cperm[(size_t)cstart[leaf] + r];
                if (q < 0 || q > INT32_MAX) return fail(H2B_ERR_INVALID, "h2b_plan_create: column index out of range");
                ix[r] = (int32_t)q;
            }
            std::memcpy(rec.data() + hdr + kFwdHead, ix, sizeof(ix));
        }
        bool warp_ok = crank[leaf] <= 32 && csize[leaf] <= 64 &&
                       (int64_t)csize[leaf] * crank[leaf] * 8 <= stage;
        int node = leaf, n = 0;
        while (true) {
            const int p = cparent[node];
            if (p < 0 || cchild[2 * p + 1] != node || !(cmask ? cmask[p] != 0 : need_c[p] != 0)) break;
            const int c0 = cchild[2 * p];
            if (n >= kMaxDepth) return fail(H2B_ERR_INVALID, "h2b_plan_create: tree deeper than 32 levels");
            rec.insert(rec.end(), {crank[c0], crank[p], ceoff[c0], ceoff[node], cxoff[c0], cxoff[p]});
            warp_ok = warp_ok && crank[c0] <= 32 && crank[p] <= 32 &&
                      8 * ((((int64_t)crank[c0] * crank[p] + 1) & ~int64_t(1)) +
                           (((int64_t)crank[node] * crank[p] + 1) & ~int64_t(1))) <= stage;
            node = p;
            ++n;
        }
        rec[hdr + 5] = n;
        rec[hdr + 6] = warp_ok ? 1 : 0;
    }
    // B/C: band records; rows per band so one band fits the TMA stage.  Near
    // bands of the owned leaves, then coupling bands of the owned clusters
    // parents first; the last band of a cluster (an empty one when it has no
    // couplings) carries the cluster's downward-step record.
    const int64_t band_base = (int64_t)rec.size();
    auto bands_to = [&](std::vector<int64_t>& out, int cols, int rows, int64_t src, int64_t gi, int64_t outo,
                        int kind) {
        int per = std::max(1, (int)(stage / (8 * std::max(cols, 1))));
        if (cols > kChunkCols) per = std::min(per, kWarps);  // chunked rows: one row per warp
        int n = 0;
        for (int r0 = 0; r0 < rows; r0 += per, ++n) {
            const int nr = std::min(per, rows - r0);
            out.insert(out.end(), {src + (int64_t)r0 * cols, cols, nr, gi, outo + r0, 0, 0, kind});
            out.insert(out.end(), kBandWords - 8, 0);
        }
        return n;
    };
    int n_cpl = 0;
    int64_t pack_len = 0;             // doubles in the packed downward-step operands
    std::vector<int64_t> pack_desc;   // per step: e_off (-1), k, k_parent, v_off (-1), size, pack offset
    // Coupling bands of cluster u: all but the last to `early`; the last one
    // (an empty band when u has no couplings) runs u's downward step and goes
    // to `late`.
    auto cluster_to = [&](std::vector<int64_t>& early, std::vector<int64_t>& late, int u) {
        if (rvoff[u] < 0 && !hasv[u]) return;  // inner cluster with v_t == 0: nothing to do
        const bool cpl = scols[u] > 0 && rrank[u] > 0;
        const int par = (rparent[u] >= 0 && hasv[rparent[u]]) ? rparent[u] : -1;  // v_parent == 0: as a root
        int64_t dw[kBandWords] = {0};  // downward-step words 5..18 of a record
        {
            const int64_t d[9] = {rrank[u], par >= 0 ? ryoff[par] : -1, par >= 0 ? rrank[par] : 0,
                                  par >= 0 ? reoff[u] : 0, ryoff[u], rvoff[u] >= 0 ? 1 : 0,
                                  rvoff[u] >= 0 ? rvoff[u] : 0, rstart[u], rsize[u]};
            dw[5] = 1;
            dw[6] = cpl ? 1 : 0;
            for (int i = 0; i < 9; ++i) dw[8 + i] = d[i];
            int dd = 0;
            for (int q = rparent[u]; q >= 0; q = rparent[q]) ++dd;
            dw[17] = dd;  // depth (diagnostics: trace)
            if (sym.on && rvoff[u] >= 0) {  // the leaf's nearfield partials (symmetric nearfield)
                dw[19] = sym.list_off[u];
                dw[20] = sym.list_n[u];
            }
            dw[23] = u;  // (plan building only)
            const int kk = rrank[u], kq = par >= 0 ? rrank[par] : 0;
            const bool lf = rvoff[u] >= 0;
            // packed operands of the step: E_u^T (kq x kk), then V_u^T (kk x |u|)
            const int64_t ne = ((int64_t)kk * kq + 1) & ~int64_t(1);
            const int64_t nv = lf ? (((int64_t)rsize[u] * kk + 1) & ~int64_t(1)) : 0;
            dw[21] = pack_len;
            dw[22] = 8 * (ne + nv);
            pack_desc.insert(pack_desc.end(), {par >= 0 ? reoff[u] : -1, kk, kq, lf ? rvoff[u] : -1, rsize[u], pack_len});
            pack_len += ne + nv;
            dw[18] = (kk <= 32 && kq <= 32 && (!lf || rsize[u] <= 64) && 8 * (ne + nv) <= stage)
                         ? 1 : 0;  // one-warp downward step
        }
        std::vector<int64_t> tmp;
        int n = cpl ? bands_to(tmp, scols[u], rrank[u], soff[u], sgoff[u], ryoff[u], kKindCpl) : 0;
        if (n == 0) {  // empty band: downward step only
            tmp.insert(tmp.end(), {0, 0, 0, 0, 0, 0, 0, kKindCpl});
            tmp.insert(tmp.end(), kBandWords - 8, 0);
            n = 1;
        }
        n_cpl += n;
        int64_t* last = tmp.data() + tmp.size() - kBandWords;
        for (int i = 5; i < kBandWords; ++i)
            if (i != 7) last[i] = dw[i];
        early.insert(early.end(), tmp.begin(), tmp.end() - kBandWords);
        late.insert(late.end(), tmp.end() - kBandWords, tmp.end());
    };
    // append `xs` with the bands of `fill` spread evenly among them
    auto interleave = [&](const std::vector<int64_t>& xs, const std::vector<int64_t>& fill) {
        const int64_t nx = (int64_t)xs.size() / kBandWords, nf = (int64_t)fill.size() / kBandWords;
        int64_t f = 0;
        for (int64_t i = 0; i < nx; ++i) {
            rec.insert(rec.end(), xs.begin() + kBandWords * i, xs.begin() + kBandWords * (i + 1));
            for (const int64_t until = (nf * (i + 1)) / nx; f < until; ++f)
                rec.insert(rec.end(), fill.begin() + kBandWords * f, fill.begin() + kBandWords * (f + 1));
        }
        rec.insert(rec.end(), fill.begin() + kBandWords * f, fill.end());
    };
    // Ticket order after the forward tasks (a task waits only on smaller
    // tickets; near bands never wait):
    //   near A1 | the leaf coupling bands except each leaf's last one (they
    //   need leaf-level x_hat only) spread over near A2 | inner-cluster
    //   coupling bands, parents first (each cluster's last band runs its
    //   downward step) spread over near B | the last band of every leaf (leaf
    //   downward step; needs every near band of its leaf).
    // The nearfield streams while the forward climb and the downward chain
    // advance.
    const double fa1 = 0.2, fa2 = 0.5;  // nearfield fractions A1, A2 (neutral within +-1 % when varied)
    std::vector<int> owned_leaves;
    for (int u : order)
        if (rvoff[u] >= 0) owned_leaves.push_back(u);
    const int nl = (int)owned_leaves.size();
    const int c1 = std::min(nl, (int)(fa1 * nl)), c2 = std::min(nl, c1 + (int)(fa2 * nl));
    std::vector<int64_t> na1, na2, nb, leaf_early, leaf_late, inner;
    int n_near = 0;
    for (int i = 0; i < nl; ++i) {
        const int u = owned_leaves[i];
        std::vector<int64_t>& dst = i < c1 ? na1 : i < c2 ? na2 : nb;
        if (sym.on) {
            dst.insert(dst.end(), sym.bands[u].begin(), sym.bands[u].end());
            n_near += (int)(sym.bands[u].size() / kBandWords);
        } else {
            n_near += bands_to(dst, dcols[u], rsize[u], doff[u], dgoff[u], rstart[u], kKindNear);
        }
    }
    for (int u : order)
        if (rvoff[u] < 0) cluster_to(inner, inner, u);
    for (int u : owned_leaves) cluster_to(leaf_early, leaf_late, u);
    rec.insert(rec.end(), na1.begin(), na1.end());
    interleave(leaf_early, na2);  // leaf products first (their x_hat are ready first)
    interleave(inner, nb);
    rec.insert(rec.end(), leaf_late.begin(), leaf_late.end());
    int64_t e_bytes_r = 0;
    for (int i = 0; i < L.r_nodes; ++i)
        if (rparent[i] >= 0 && reoff[i] >= 0)
            e_bytes_r = std::max<int64_t>(e_bytes_r, 8 * (reoff[i] + (int64_t)rrank[i] * rrank[rparent[i]]));

    h2b_plan* p = new (std::nothrow) h2b_plan();
    if (!p) return fail(H2B_ERR_INVALID, "h2b_plan_create: out of host memory");
    p->L = L;
    p->n_near = n_near;
    p->n_cpl = n_cpl;
    p->band_base = band_base;
    {
        int64_t m = 0;
        for (int i = 0; i < L.r_nodes; ++i)
            if (rvoff[i] >= 0) m = std::max<int64_t>(m, 4 * (dgoff[i] + dcols[i]));
        p->dgidx_bytes = sym.on ? 4 * (int64_t)sym.gsym.size() : m;
    }
    p->max_cols = maxcols;
    p->vec_len = vec_len;
    p->smem = smem;
    p->stage_bytes = stage;
    p->e_bytes_r = e_bytes_r;
    H2B_CUDA_TRY(cudaGetDevice(&p->device));
    H2B_CUDA_TRY(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming));
    auto alloc = [](void** ptr, size_t bytes) { return cudaMalloc(ptr, bytes ? bytes : 16); };
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->xhat), 16 * (size_t)L.xhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ycpl), 16 * (size_t)L.yhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->yfin), 16 * (size_t)L.yhat_len));
    H2B_CUDA_TRY(cudaMemset(p->yfin, 0, 16 * (size_t)L.yhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ynear), 16 * (size_t)L.n_rows));
    H2B_CUDA_TRY(cudaMemset(p->xhat, 0, 16 * (size_t)L.xhat_len));
    H2B_CUDA_TRY(cudaMemset(p->ycpl, 0, 16 * (size_t)L.yhat_len));
    H2B_CUDA_TRY(cudaMemset(p->ynear, 0, 16 * (size_t)L.n_rows));
    // ticket counters: [0] matvec launches, [3] forward launches of the x_hat
    // exchange ([1], [2] unused)
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ctrl), 4 * sizeof(unsigned long long)));
    H2B_CUDA_TRY(cudaMemset(p->ctrl, 0, 4 * sizeof(unsigned long long)));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->rec), sizeof(int64_t) * std::max<size_t>(1, rec.size())));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->fwd_off), sizeof(int64_t) * std::max<size_t>(1, fwd_off.size())));
    if (!rec.empty())
        H2B_CUDA_TRY(cudaMemcpy(p->rec, rec.data(), sizeof(int64_t) * rec.size(), cudaMemcpyHostToDevice));
    if (!fwd_off.empty())
        H2B_CUDA_TRY(cudaMemcpy(p->fwd_off, fwd_off.data(), sizeof(int64_t) * fwd_off.size(), cudaMemcpyHostToDevice));
    p->n_fwd = (int)fwd_off.size();
    {
        // the downward steps' operands, transposed once (plan-owned copy)
        H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->dpack), 8 * (size_t)pack_len));
        H2B_CUDA_TRY(cudaMemset(p->dpack, 0, 8 * (size_t)std::max<int64_t>(pack_len, 2)));
        const int64_t nd = (int64_t)pack_desc.size() / 6;
        if (nd > 0) {
            int64_t* d_desc = nullptr;
            H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&d_desc), 8 * pack_desc.size()));
            H2B_CUDA_TRY(cudaMemcpy(d_desc, pack_desc.data(), 8 * pack_desc.size(), cudaMemcpyHostToDevice));
            k_pack_descent<<<(unsigned)nd, 128>>>(L.r_E, L.r_V, d_desc, p->dpack);
            cudaError_t e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            cudaFree(d_desc);
            H2B_CUDA_TRY(e);
        }
    }
    if (cmask) {
        p->xmode = true;
        H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->xhat_f), 16 * (size_t)L.xhat_len));
        H2B_CUDA_TRY(cudaMemset(p->xhat_f, 0, 16 * (size_t)L.xhat_len));
        H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->span_val), 8 * (size_t)L.xhat_len));
        std::vector<int32_t> own;
        std::vector<int64_t> own_off;
        int64_t o = 0;
        for (int u = 0; u < L.c_nodes; ++u)
            if (cmask[u]) {
                own.push_back(u);
                own_off.push_back(o);
                o += crank[u];
            }
        p->n_own = (int)own.size();
        p->send_len = o;
        H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->d_own), 4 * std::max<size_t>(1, own.size())));
        H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->d_own_off), 8 * std::max<size_t>(1, own.size())));
        if (!own.empty()) {
            H2B_CUDA_TRY(cudaMemcpy(p->d_own, own.data(), 4 * own.size(), cudaMemcpyHostToDevice));
            H2B_CUDA_TRY(cudaMemcpy(p->d_own_off, own_off.data(), 8 * own.size(), cudaMemcpyHostToDevice));
        }
    }
    {
        // the attribute belongs to the kernel, not the plan: only ever raise it
        // (a later plan with less shared memory must not break an earlier one)
        static int smem_set[64] = {0};
        int& cur = smem_set[p->device & 63];
        if (p->smem > cur) {
            H2B_CUDA_TRY(cudaFuncSetAttribute(k_matvec<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, p->smem));
            H2B_CUDA_TRY(cudaFuncSetAttribute(k_matvec<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, p->smem));
            cur = p->smem;
        }
    }
    p->trace = nullptr;
    if (const char* tr = getenv("H2B_TRACE")) {
        if (tr[0] == '1') {
            const size_t n = (size_t)(fwd_off.size() + n_near + n_cpl) * 8;
            H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&p->trace), n * sizeof(unsigned long long)));
            H2B_CUDA_TRY(cudaMemset(p->trace, 0, n * sizeof(unsigned long long)));
        }
    }
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->dx), sizeof(double) * L.n_cols));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->dy), sizeof(double) * L.n_rows));
    p->dsym = nullptr;
    p->gsym = nullptr;
    p->ppart = nullptr;
    p->nsum = nullptr;
    p->near_bytes = 0;
    p->cpl_bytes = 0;
    p->ppart_len = 0;
    for (int u = 0; u < L.r_nodes; ++u) {
        if (rvoff[u] >= 0) p->near_bytes += 8 * (int64_t)rsize[u] * dcols[u];
        p->cpl_bytes += 8 * (int64_t)rrank[u] * scols[u];
    }
    if (sym.on) {
        // symmetric storage needs the operator's blocks symmetric bit for bit
        // (checked on the device); then the upper blocks are packed into the
        // column panels the tasks stream
        auto check = [&](const double* base, const std::vector<int64_t>& jobs, int& bad) -> int {
            int64_t* dj = nullptr;
            int* db = nullptr;
            H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&dj), 8 * std::max<size_t>(jobs.size(), 1)));
            H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&db), sizeof(int)));
            H2B_CUDA_TRY(cudaMemset(db, 0, sizeof(int)));
            H2B_CUDA_TRY(cudaMemcpy(dj, jobs.data(), 8 * jobs.size(), cudaMemcpyHostToDevice));
            if (!jobs.empty()) k_sym_check<<<(unsigned)(jobs.size() / 6), 256>>>(base, dj, db);
            H2B_CUDA_TRY(cudaGetLastError());
            H2B_CUDA_TRY(cudaMemcpy(&bad, db, sizeof(int), cudaMemcpyDeviceToHost));
            cudaFree(dj);
            cudaFree(db);
            return 0;
        };
        auto pack = [&](const double* base, const std::vector<int64_t>& jobs, const std::vector<int32_t>& srccol,
                        int64_t len, double** dst) -> int {
            int64_t* dj = nullptr;
            int32_t* ds = nullptr;
            H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&dj), 8 * std::max<size_t>(jobs.size(), 1)));
            H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&ds), 4 * std::max<size_t>(srccol.size(), 1)));
            H2B_CUDA_TRY(cudaMemcpy(dj, jobs.data(), 8 * jobs.size(), cudaMemcpyHostToDevice));
            H2B_CUDA_TRY(cudaMemcpy(ds, srccol.data(), 4 * srccol.size(), cudaMemcpyHostToDevice));
            H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(dst), 8 * (size_t)std::max<int64_t>(len, 2)));
            H2B_CUDA_TRY(cudaMemset(*dst, 0, 8 * (size_t)std::max<int64_t>(len, 2)));
            if (!jobs.empty()) k_sym_pack<<<(unsigned)(jobs.size() / 6), 256>>>(base, dj, ds, *dst);
            H2B_CUDA_TRY(cudaGetLastError());
            H2B_CUDA_TRY(cudaDeviceSynchronize());
            cudaFree(dj);
            cudaFree(ds);
            return 0;
        };
        auto upload = [&](const auto& v, auto** dst) -> int {
            using T = typename std::decay_t<decltype(v)>::value_type;
            H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(dst), sizeof(T) * std::max<size_t>(v.size(), 1)));
            if (!v.empty()) H2B_CUDA_TRY(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
            return 0;
        };
        int bad_near = 0;
        if (int rc = check(L.D, sym.check, bad_near)) return rc;
        if (bad_near) {
            // not symmetric: stream every block
            h2b_plan_destroy(p);
            return plan_create(layout, out, sym_flags & ~kSymNear);
        }
        if (int rc = pack(L.D, sym.pack, sym.srccol, sym.dsym_len, &p->dsym)) return rc;
        if (int rc = upload(sym.gsym, &p->gsym)) return rc;
        p->near_bytes = sym.near_bytes;
        p->ppart_len = sym.ppart_len;
        H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ppart), 16 * (size_t)std::max<int64_t>(p->ppart_len, 1)));
        H2B_CUDA_TRY(cudaMemset(p->ppart, 0, 16 * (size_t)std::max<int64_t>(p->ppart_len, 1)));
        if (int rc = upload(sym.nsum, &p->nsum)) return rc;
    }
    *out = p;
    return ok();
}
}  // namespace

extern "C" int h2b_plan_create(const h2b_layout* layout, h2b_plan** out) {
    return plan_create(layout, out, kSymNear);
}

#ifdef H2B_LL_TIMEOUT
extern "C" int h2b_debug_stuck(h2b_plan* p, unsigned long long* out) {
    unsigned long long h[4];
    H2B_CUDA_TRY(cudaMemcpyFromSymbol(h, g_ll_stuck, sizeof(h)));
    out[0] = h[0];
    out[1] = h[1];
    out[2] = h[2];
    out[3] = reinterpret_cast<unsigned long long>(p->xhat);
    out[4] = reinterpret_cast<unsigned long long>(p->ycpl);
    out[5] = reinterpret_cast<unsigned long long>(p->yfin);
    out[6] = reinterpret_cast<unsigned long long>(p->ynear);
    out[7] = h[3];  // the word found at the abandoned address
    unsigned long long mb[4];
    H2B_CUDA_TRY(cudaMemcpyFromSymbol(mb, g_mbar_stuck, sizeof(mb)));
    out[8] = mb[0];
    out[9] = mb[1];
    out[10] = mb[2];  // abandoned mbarrier waits
    out[11] = mb[3];  // longest mbarrier wait (ns)
    return 0;
}
#endif

extern "C" int h2b_plan_destroy(h2b_plan* p) {
    if (!p) return ok();
    if (p->hx) cudaFreeHost(p->hx);
    void* bufs[] = {p->xhat, p->ycpl, p->yfin, p->ynear, p->ctrl, p->rec,  p->fwd_off, p->dx,
                    p->dy,   p->trace, p->dsym, p->dpack,  p->gsym, p->ppart, p->nsum, p->xgath,
                    p->xhat_f, p->d_own, p->d_own_off, p->d_imp, p->d_imp_src, p->d_span, p->span_val};
    for (void* q : bufs)
        if (q) cudaFree(q);
    if (p->done) cudaEventDestroy(p->done);
    delete p;
    return ok();
}

namespace {
// mode 0: the plan's full task list; 1: forward tasks only (x_hat exchange,
// into xhat_f); 2: bands only (x_hat imported)
int launch_matvec(h2b_plan* p, const double* d_x, double* y, cudaStream_t st, int mode = 0) {
    // (caller holds p->mu) order after the plan's previous launch if that was
    // on another stream
    if (p->launched && p->last != st) H2B_CUDA_TRY(cudaStreamWaitEvent(st, p->done, 0));
    KArgs a;
    a.L = p->L;
    a.rec = p->rec;
    a.fwd_off = p->fwd_off;
    a.band_base = p->band_base;
    a.band_bytes = 8 * (int64_t)kBandWords * (p->n_near + p->n_cpl);
    a.dgidx_bytes = p->dgidx_bytes;
    // The forward tasks pull the band records and nearfield gather lists into
    // L2 up front only when these are small: at config 1 (2 MB) that saves 4 %,
    // at configs 2 and 3 (70 / 190 MB against a 126 MB L2 that also holds x,
    // x_hat and the partial vectors) it costs 2 % (same-box A/B).
    if (a.band_bytes + a.dgidx_bytes > kUpfrontMax) a.band_bytes = a.dgidx_bytes = 0;
    a.n_near = p->n_near;
    a.n_cpl = p->n_cpl;
    a.max_cols = p->max_cols;
    a.vec_len = p->vec_len;
    a.stage_bytes = p->stage_bytes;
    a.e_bytes_r = p->e_bytes_r;
    a.xhat = p->xhat;
    a.ycpl = p->ycpl;
    a.yfin = p->yfin;
    a.ynear = p->ynear;
    a.ctrl = p->ctrl;
    a.trace = p->trace;
    a.dsym = p->dsym;
    a.gsym = p->gsym;
    a.ppart = p->ppart;
    a.nsum = p->nsum;
    a.dpack = p->dpack;
    a.n_fwd = p->n_fwd;
    if (mode == 1) {
        a.n_near = a.n_cpl = 0;
        a.xhat = p->xhat_f;
        a.ctrl = p->ctrl + 3;
    } else if (mode == 2) {
        a.n_fwd = 0;
    }
    const int grid = a.n_fwd + a.n_near + a.n_cpl;
    if (p->trace)
        k_matvec<true><<<grid, kThreads, p->smem, st>>>(a, d_x, y);  // diagnostic timeline (H2B_TRACE=1 at plan creation)
    else
        k_matvec<false><<<grid, kThreads, p->smem, st>>>(a, d_x, y);
    H2B_CUDA_TRY(cudaGetLastError());
    H2B_CUDA_TRY(cudaEventRecord(p->done, st));
    p->last = st;
    p->launched = true;
    return ok();
}

}  // namespace

extern "C" int h2b_matvec(h2b_plan* p, const double* d_x, double* d_y, void* stream) {
    if (!p || !d_x || !d_y) return fail(H2B_ERR_INVALID, "h2b_matvec: null pointer");
    if (p->xmode) return fail(H2B_ERR_INVALID, "h2b_matvec: x_hat-exchange plan (use h2b_xhat_forward / h2b_xhat_main)");
    std::lock_guard<std::mutex> g(p->mu);
    return launch_matvec(p, d_x, d_y, as_stream(stream));
}

namespace {
// A pageable x of config 3 is 16.8 MB: the driver's staged host-to-device copy
// moves it at the speed of one core's memcpy (~1 ms), a third of the matvec.
// StagePool copies it into the plan's page-locked staging buffer with three
// persistent host threads and the caller, piece by piece, while the calling thread hands every
// finished piece to the copy engine (cudaMemcpyAsync): memcpy and DMA overlap
// and the memcpy runs on several cores.  (Threads spawned per call cost more
// than they saved; in-kernel polling of arrival flags was slower still.)
class StagePool {
public:
    static constexpr size_t kPiece = size_t(1) << 20;
    static StagePool& get() {
        static StagePool pool;
        return pool;
    }
    // false: not usable here (forked child, thread start failed): use the plain copy
    bool usable() { return pid_ == getpid() && !th_->empty(); }
    std::mutex use;  // one staged copy at a time

    // dst (page-locked) <- src, then DMA to dev piece by piece on st
    cudaError_t copy(double* dev, double* dst, const double* src, size_t bytes, cudaStream_t st) {
        const size_t np = (bytes + kPiece - 1) / kPiece;
        {
            // workers become active under this lock only: with none active the
            // job may change (a straggler of the last job finds no piece left)
            std::unique_lock<std::mutex> g(m_);
            while (active_.load(std::memory_order_acquire) != 0) {
                g.unlock();
                std::this_thread::yield();
                g.lock();
            }
            if (done_.size() < np) done_ = std::vector<std::atomic<uint32_t>>(np);
            dst_ = reinterpret_cast<char*>(dst);
            src_ = reinterpret_cast<const char*>(src);
            bytes_ = bytes;
            np_ = np;
            next_.store(0, std::memory_order_relaxed);
            ++seq_;
        }
        cv_.notify_all();
        const uint32_t seq = seq_;
        for (size_t k = 0; k < np; ++k) {
            while (done_[k].load(std::memory_order_acquire) != seq) {
                if (!work_one(seq)) std::this_thread::yield();
            }
            const size_t o = k * kPiece, n = std::min(kPiece, bytes - o);
            const cudaError_t e = cudaMemcpyAsync(reinterpret_cast<char*>(dev) + o, dst_ + o, n, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) {
                // let the remaining pieces finish before the buffers go away
                for (size_t j = k + 1; j < np; ++j)
                    while (done_[j].load(std::memory_order_acquire) != seq)
                        if (!work_one(seq)) std::this_thread::yield();
                return e;
            }
        }
        return cudaSuccess;
    }

private:
    StagePool() : pid_(getpid()), th_(new std::vector<std::thread>()) {
        const unsigned hw = std::thread::hardware_concurrency();
        // three workers beside the calling thread.  Per call at config 3: one
        // box 3.66 ms against 4.15 ms with the driver's staged copy; on another
        // (virtualised, slow thread wake-ups) 1 / 3 / 5 / 7 / 11 workers gave
        // 3.93 / 4.08 / 4.44 / 4.45 / 4.90 ms against 4.11 ms: never worse with
        // three, more threads lose to wake-up latency and stragglers
        const int nt = (int)std::min(3u, hw > 1 ? hw - 1 : 0u);
        try {
            for (int i = 0; i < nt; ++i) th_->emplace_back([this] { run(); });
        } catch (...) {
        }
    }
    ~StagePool() {
        if (pid_ != getpid()) return;  // forked child: the threads are not ours (their handles stay untouched)
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : *th_) t.join();
        delete th_;
    }
    bool work_one(uint32_t seq) {
        const size_t k = next_.fetch_add(1, std::memory_order_relaxed);
        if (k >= np_) return false;
        const size_t o = k * kPiece;
        std::memcpy(dst_ + o, src_ + o, std::min(kPiece, bytes_ - o));
        done_[k].store(seq, std::memory_order_release);
        return true;
    }
    void run() {
        uint32_t seen = 0;
        for (;;) {
            uint32_t seq;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || seq_ != seen; });
                if (stop_) return;
                seen = seq = seq_;
                active_.fetch_add(1, std::memory_order_acq_rel);
            }
            while (work_one(seq)) {
            }
            active_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    pid_t pid_;
    std::vector<std::thread>* th_;
    std::mutex m_;
    std::condition_variable cv_;
    bool stop_ = false;
    uint32_t seq_ = 0;
    std::atomic<int> active_{0};
    std::atomic<size_t> next_{0};
    size_t np_ = 0, bytes_ = 0;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    std::vector<std::atomic<uint32_t>> done_;
};

bool page_locked(const void* h) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
}  // namespace

// Host vectors: one stream-ordered copy each way around the launch (a
// page-locked buffer by DMA; a large pageable x through StagePool, a small one
// or a pageable y through the driver's staged copy), then a stream
// synchronise.  Measured against the round's earlier design -- x read from
// mapped host memory by copy tasks inside the kernel, y written to mapped host
// memory by its last tasks -- the copy engines win from config 2 up (config 3,
// pinned vectors: 3.46 vs 3.82 ms) and cost 3 us at config 1 (76 vs 73 us).
extern "C" int h2b_matvec_host(h2b_plan* p, const double* h_x, double* h_y, void* stream) {
    if (!p || !h_x || !h_y) return fail(H2B_ERR_INVALID, "h2b_matvec_host: null pointer");
    if (p->xmode) return fail(H2B_ERR_INVALID, "h2b_matvec_host: x_hat-exchange plan");
    std::lock_guard<std::mutex> g(p->mu);
    cudaStream_t st = as_stream(stream);
    if (p->launched && p->last != st) H2B_CUDA_TRY(cudaStreamWaitEvent(st, p->done, 0));
    const size_t xbytes = sizeof(double) * p->L.n_cols;
    bool staged = false;
    if (xbytes >= 4 * StagePool::kPiece && !page_locked(h_x)) {
        StagePool& pool = StagePool::get();
        if (pool.usable()) {
            if (!p->hx) H2B_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&p->hx), xbytes));
            std::lock_guard<std::mutex> u(pool.use);
            H2B_CUDA_TRY(pool.copy(p->dx, p->hx, h_x, xbytes, st));
            staged = true;
        }
    }
    if (!staged) H2B_CUDA_TRY(cudaMemcpyAsync(p->dx, h_x, xbytes, cudaMemcpyHostToDevice, st));
    if (int rc = launch_matvec(p, p->dx, p->dy, st)) return rc;
    H2B_CUDA_TRY(cudaMemcpyAsync(h_y, p->dy, sizeof(double) * p->L.n_rows, cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    return ok();
}

extern "C" int h2b_plan_set_comm(h2b_plan* p, void* comm, int rank, int nranks, int64_t chunk) {
    if (!p || !comm || nranks < 1 || rank < 0 || rank >= nranks || chunk < 1)
        return fail(H2B_ERR_INVALID, "h2b_plan_set_comm: bad argument");
    if ((int64_t)nranks * chunk < p->L.n_cols)
        return fail(H2B_ERR_INVALID, "h2b_plan_set_comm: gathered x shorter than the plan's columns");
    if (!nccl_api()) return fail(H2B_ERR_INVALID, "h2b_plan_set_comm: libnccl.so.2 not found");
    std::lock_guard<std::mutex> g(p->mu);
    if (p->xgath) {
        cudaFree(p->xgath);
        p->xgath = nullptr;
    }
    H2B_CUDA_TRY(cudaSetDevice(p->device));
    H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&p->xgath), sizeof(double) * nranks * chunk));
    p->comm = comm;
    p->comm_rank = rank;
    p->comm_size = nranks;
    p->comm_chunk = chunk;
    return ok();
}

extern "C" int h2b_matvec_sharded(h2b_plan* p, const double* d_x_local, double* d_y_local, void* stream) {
    if (!p || !d_x_local || !d_y_local) return fail(H2B_ERR_INVALID, "h2b_matvec_sharded: null pointer");
    if (!p->comm) return fail(H2B_ERR_INVALID, "h2b_matvec_sharded: no communicator (h2b_plan_set_comm)");
    std::lock_guard<std::mutex> g(p->mu);
    cudaStream_t st = as_stream(stream);
    const NcclApi* api = nccl_api();
    if (p->launched && p->last != st) H2B_CUDA_TRY(cudaStreamWaitEvent(st, p->done, 0));
    const ncclResult_t r = api->all_gather(d_x_local, p->xgath, (size_t)p->comm_chunk, ncclFloat64,
                                           static_cast<ncclComm_t>(p->comm), st);
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllGather");
    return launch_matvec(p, p->xgath, d_y_local, st);
}

extern "C" int h2b_plan_create_xhat(const h2b_layout* layout, const int8_t* h_cmask, h2b_plan** out) {
    if (!h_cmask) return fail(H2B_ERR_INVALID, "h2b_plan_create_xhat: null mask");
    return plan_create(layout, out, kSymNear, h_cmask);
}

extern "C" int h2b_xhat_info(h2b_plan* p, int64_t* h_out) {
    if (!p || !h_out) return fail(H2B_ERR_INVALID, "h2b_xhat_info: null pointer");
    h_out[0] = p->n_own;
    h_out[1] = p->send_len;
    h_out[2] = p->n_fwd;
    h_out[3] = p->n_imp;
    h_out[4] = p->span_level_off.empty() ? 0 : p->span_level_off.back();
    return ok();
}

extern "C" int h2b_xhat_set_import(h2b_plan* p, const int64_t* h_src) {
    if (!p || !h_src) return fail(H2B_ERR_INVALID, "h2b_xhat_set_import: null pointer");
    if (!p->xmode) return fail(H2B_ERR_INVALID, "h2b_xhat_set_import: plan not created for the x_hat exchange");
    std::lock_guard<std::mutex> g(p->mu);
    const h2b_layout& L = p->L;
    std::vector<int32_t> cparent, cchild;
    H2B_CUDA_TRY(fetch(L.c_parent, L.c_nodes, cparent));
    H2B_CUDA_TRY(fetch(L.c_child, 2 * (int64_t)L.c_nodes, cchild));
    std::vector<int32_t> imp, span;
    std::vector<int64_t> src;
    std::vector<int> depth(L.c_nodes, 0);
    for (int u = 0; u < L.c_nodes; ++u) {
        for (int q = cparent[u]; q >= 0; q = cparent[q]) ++depth[u];
        if (h_src[u] >= 0) {
            imp.push_back(u);
            src.push_back(h_src[u]);
        } else {
            if (cchild[2 * u] < 0) return fail(H2B_ERR_INVALID, "h2b_xhat_set_import: a leaf without coefficients");
            span.push_back(u);
        }
    }
    // spanning clusters deepest level first (children before parents)
    std::stable_sort(span.begin(), span.end(), [&](int a, int b) { return depth[a] > depth[b]; });
    p->span_level_off.assign(1, 0);
    for (size_t i = 0; i < span.size(); ++i)
        if (i + 1 == span.size() || depth[span[i + 1]] != depth[span[i]]) p->span_level_off.push_back((int64_t)i + 1);
    for (void* q : {(void*)p->d_imp, (void*)p->d_imp_src, (void*)p->d_span})
        if (q) cudaFree(q);
    H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&p->d_imp), 4 * std::max<size_t>(1, imp.size())));
    H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&p->d_imp_src), 8 * std::max<size_t>(1, imp.size())));
    H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&p->d_span), 4 * std::max<size_t>(1, span.size())));
    if (!imp.empty()) {
        H2B_CUDA_TRY(cudaMemcpy(p->d_imp, imp.data(), 4 * imp.size(), cudaMemcpyHostToDevice));
        H2B_CUDA_TRY(cudaMemcpy(p->d_imp_src, src.data(), 8 * src.size(), cudaMemcpyHostToDevice));
    }
    if (!span.empty()) H2B_CUDA_TRY(cudaMemcpy(p->d_span, span.data(), 4 * span.size(), cudaMemcpyHostToDevice));
    p->n_imp = (int)imp.size();
    return ok();
}

extern "C" int h2b_xhat_forward(h2b_plan* p, const double* d_x, double* d_send, void* stream) {
    if (!p || !d_x || !d_send) return fail(H2B_ERR_INVALID, "h2b_xhat_forward: null pointer");
    if (!p->xmode) return fail(H2B_ERR_INVALID, "h2b_xhat_forward: plan not created for the x_hat exchange");
    std::lock_guard<std::mutex> g(p->mu);
    cudaStream_t st = as_stream(stream);
    const uint32_t epoch = 2u * (uint32_t)p->n_f_launches + 1u;
    if (p->n_fwd > 0) {
        if (int rc = launch_matvec(p, d_x, nullptr, st, 1)) return rc;
    }
    ++p->n_f_launches;
    if (p->n_own > 0) {
        k_xhat_pack<<<(unsigned)((32 * (int64_t)p->n_own + 255) / 256), 256, 0, st>>>(
            p->L, p->xhat_f, epoch, p->d_own, p->d_own_off, p->n_own, d_send);
        H2B_CUDA_TRY(cudaGetLastError());
    }
    return ok();
}

extern "C" int h2b_xhat_main(h2b_plan* p, const double* d_x, const double* d_recv, double* d_y, void* stream) {
    if (!p || !d_x || !d_recv || !d_y) return fail(H2B_ERR_INVALID, "h2b_xhat_main: null pointer");
    if (!p->xmode || p->span_level_off.empty())
        return fail(H2B_ERR_INVALID, "h2b_xhat_main: x_hat exchange not set up (h2b_xhat_set_import)");
    std::lock_guard<std::mutex> g(p->mu);
    cudaStream_t st = as_stream(stream);
    if (p->launched && p->last != st) H2B_CUDA_TRY(cudaStreamWaitEvent(st, p->done, 0));
    const uint32_t epoch = 2u * (uint32_t)p->n_m_launches + 1u;  // the bands launch below
    if (p->n_imp > 0) {
        k_xhat_import<<<(unsigned)((32 * (int64_t)p->n_imp + 255) / 256), 256, 0, st>>>(
            p->L, d_recv, p->d_imp, p->d_imp_src, p->n_imp, p->xhat, epoch, p->span_val);
        H2B_CUDA_TRY(cudaGetLastError());
    }
    const int smem = p->stage_bytes + 8 * (4 * p->vec_len + kWarps * 64);
    {
        static int set[64] = {0};
        int& cur = set[p->device & 63];
        if (smem > cur) {
            H2B_CUDA_TRY(cudaFuncSetAttribute(k_xhat_climb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            cur = smem;
        }
    }
    for (size_t l = 0; l + 1 < p->span_level_off.size(); ++l) {
        const int64_t a = p->span_level_off[l], b = p->span_level_off[l + 1];
        k_xhat_climb<<<(unsigned)(b - a), kThreads, smem, st>>>(p->L, p->d_span + a, p->stage_bytes, p->vec_len,
                                                                 p->span_val, p->xhat, epoch);
        H2B_CUDA_TRY(cudaGetLastError());
    }
    if (int rc = launch_matvec(p, d_x, d_y, st, 2)) return rc;
    ++p->n_m_launches;
    return ok();
}

// Diagnostics: the per-CTA timeline of the last matvec when the plan was
// created with H2B_TRACE=1: 8 words per ticket (start ns, end ns, SM id, 5
// phase marks), then the task-range boundaries [near, coupling, leaf, total,
// total].
extern "C" int h2b_plan_trace(h2b_plan* p, unsigned long long* h_out, int64_t cap) {
    if (!p || !h_out) return fail(H2B_ERR_INVALID, "h2b_plan_trace: null pointer");
    if (!p->trace) return fail(H2B_ERR_INVALID, "h2b_plan_trace: plan created without H2B_TRACE=1");
    const int64_t n = (int64_t)(p->n_fwd + p->n_near + p->n_cpl);
    if (cap < 8 * n + 5) return fail(H2B_ERR_CAPACITY, "h2b_plan_trace: buffer too small");
    H2B_CUDA_TRY(cudaMemcpy(h_out, p->trace, sizeof(unsigned long long) * 8 * n, cudaMemcpyDeviceToHost));
    h_out[8 * n] = p->n_fwd;
    h_out[8 * n + 1] = p->n_fwd + p->n_near;
    h_out[8 * n + 2] = n;
    h_out[8 * n + 3] = n;
    h_out[8 * n + 4] = n;
    return ok();
}

// Plan facts: [0] symmetric nearfield in use (0/1), [1] nearfield bytes one
// matvec streams, [2] nearfield tasks, [3] coupling tasks, [4] bytes of the
// symmetric partial vectors (LL form), [5] symmetric couplings in use (0/1),
// [6] coupling bytes one matvec streams, [7] TMA stage bytes per CTA,
// [8] dynamic shared memory per CTA.
extern "C" int h2b_plan_info(h2b_plan* p, int64_t* h_out) {
    if (!p || !h_out) return fail(H2B_ERR_INVALID, "h2b_plan_info: null pointer");
    h_out[0] = p->dsym != nullptr;
    h_out[1] = p->near_bytes;
    h_out[2] = p->n_near;
    h_out[3] = p->n_cpl;
    h_out[4] = p->ppart_len * 16;
    h_out[5] = 0;  // (symmetric coupling panels: measured slower, removed)
    h_out[6] = p->cpl_bytes;
    h_out[7] = p->stage_bytes;
    h_out[8] = p->smem;
    return ok();
}

extern "C" int h2b_diagonal(h2b_plan* p, double* d_diag, void* stream) {
    if (!p || !d_diag) return fail(H2B_ERR_INVALID, "h2b_diagonal: null pointer");
    if (p->L.n_rows != p->L.n_cols) return fail(H2B_ERR_INVALID, "diagonal extraction requires a square operator");
    cudaStream_t st = as_stream(stream);
    const int n = p->L.owned ? p->L.n_owned : p->L.r_nodes;
    if (n > 0) k_diagonal<<<(n + 127) / 128, 128, 0, st>>>(p->L, d_diag);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}
