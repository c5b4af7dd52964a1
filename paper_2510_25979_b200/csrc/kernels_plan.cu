// kernels_plan.cu — owner-affinity placement on the device (multi-GPU; the host function
// attncache_affinity_plan in attncache.cu defines the plan, this kernel reproduces it bit for bit and
// derives one rank's relocation lists, so the placement needs no host round trip beyond a few counts).
//
//   hits:   assign[b] = the rank whose shard [sb[r], sb[r+1]) holds idx[b] (the last such r: empty shards are
//           skipped), load[r] += hit_cost per hit
//   misses: ascending b, each on the least-loaded rank (lowest rank on ties), load[r] += miss_cost
//
// One CTA of 1024 threads.  The per-rank sums are sequential additions of one constant, as on the host,
// so every comparison and every load is identical to the host's.  Misses are placed by warp 0, lane r
// holding rank r's load (world <= 32): the current minimum takes misses one after another for as long as
// it stays the minimum (one fp64 add each), and a warp argmin re-elects it only when it changes.
// Then this rank's lists: loc (batch positions placed here, ascending) with their idx / hit, send_order
// (this rank's home rows stably sorted by destination) and counts = [send_n | recv_n | n_loc].
#include "kernels.cuh"

namespace ac {

namespace {

constexpr int kPlanThreads = 1024;

// Order-preserving compaction of the positions b in [lo, hi) with pred(b) into out[base + ...]; returns the
// number written.  All threads of the CTA call it (chunks of kPlanThreads; warp ballots + a CTA prefix).
template <typename Pred, typename Emit>
__device__ int64_t compact(int64_t lo, int64_t hi, Pred pred, Emit emit, int *warp_cnt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t written = 0;
    for (int64_t c0 = lo; c0 < hi; c0 += kPlanThreads) {
        const int64_t b = c0 + threadIdx.x;
        const bool p = b < hi && pred(b);
        const unsigned m = __ballot_sync(0xffffffffu, p);
        if (lane == 0) warp_cnt[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < kPlanThreads / 32; ++w) {
            const int cnt = warp_cnt[w];
            before += w < warp ? cnt : 0;
            total += cnt;
        }
        if (p) emit(written + before + __popc(m & ((1u << lane) - 1u)), b);
        written += total;
        __syncthreads();
    }
    return written;
}

__global__ void __launch_bounds__(kPlanThreads, 1)
    affinity_plan_kernel(const int64_t *__restrict__ idx, const uint8_t *__restrict__ hit, int64_t n, PlanArgs a,
                         int32_t *assign, double *load, int64_t *miss_list, int64_t *loc, int64_t *idx_loc,
                         uint8_t *hit_loc, int64_t *send_order, int32_t *counts) {
    __shared__ int64_t sb[kPlanMaxWorld + 1];
    __shared__ int hits_per_rank[kPlanMaxWorld];
    __shared__ int warp_cnt[kPlanThreads / 32];
    const int world = a.world;
    if (threadIdx.x <= world) sb[threadIdx.x] = a.shard_begins[threadIdx.x];
    if (threadIdx.x < kPlanMaxWorld) hits_per_rank[threadIdx.x] = 0;
    __syncthreads();
    // hits: the owner (binary search for the last r with sb[r] <= e)
    for (int64_t b = threadIdx.x; b < n; b += kPlanThreads) {
        if (!hit[b]) continue;
        const int64_t e = idx[b];
        int lo = 0, hi = world - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (sb[mid] <= e) lo = mid; else hi = mid - 1;
        }
        assign[b] = lo;
        atomicAdd(&hits_per_rank[lo], 1);
    }
    // misses in ascending batch order
    const int64_t n_miss = compact(0, n, [&](int64_t b) { return hit[b] == 0; },
                                   [&](int64_t at, int64_t b) { miss_list[at] = b; }, warp_cnt);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int r = threadIdx.x;
        double acc = 0.0;
        if (r < world)
            for (int k = 0; k < hits_per_rank[r]; ++k) acc += a.hit_cost;
        int64_t next = 0;
        while (next < n_miss) {
            // argmin and runner-up of (load, rank) over the live lanes
            double v1 = r < world ? acc : INFINITY;
            int r1 = r < world ? r : 1 << 30;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v1, o);
                const int orr = __shfl_xor_sync(0xffffffffu, r1, o);
                if (ov < v1 || (ov == v1 && orr < r1)) v1 = ov, r1 = orr;
            }
            double v2 = (r < world && r != r1) ? acc : INFINITY;
            int r2 = (r < world && r != r1) ? r : 1 << 30;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v2, o);
                const int orr = __shfl_xor_sync(0xffffffffu, r2, o);
                if (ov < v2 || (ov == v2 && orr < r2)) v2 = ov, r2 = orr;
            }
            int64_t taken = 0;
            if (r == r1) {
                // r1 takes misses while it stays the minimum: (acc, r1) < (v2, r2)
                do {
                    assign[miss_list[next + taken]] = r1;
                    acc += a.miss_cost;
                    ++taken;
                } while (next + taken < n_miss && (acc < v2 || (acc == v2 && r1 < r2)));
            }
            next += __shfl_sync(0xffffffffu, taken, r1 & 31);
        }
        if (r < world) load[r] = acc;
    }
    __syncthreads();
    // this rank's lists
    const int me = a.rank;
    const int64_t n_loc = compact(0, n, [&](int64_t b) { return assign[b] == me; },
                                  [&](int64_t at, int64_t b) {
                                      loc[at] = b;
                                      idx_loc[at] = hit[b] ? idx[b] : 0;
                                      hit_loc[at] = hit[b];
                                  },
                                  warp_cnt);
    const int64_t h0 = a.home_begins[me], h1 = a.home_begins[me + 1];
    int64_t sent = 0;
    for (int d = 0; d < world; ++d) {
        const int64_t c = compact(h0, h1, [&](int64_t b) { return assign[b] == d; },
                                  [&](int64_t at, int64_t b) { send_order[sent + at] = b - h0; }, warp_cnt);
        if (threadIdx.x == 0) counts[d] = (int32_t)c;
        sent += c;
    }
    for (int s = 0; s < world; ++s) {
        const int64_t c = compact(a.home_begins[s], a.home_begins[s + 1], [&](int64_t b) { return assign[b] == me; },
                                  [&](int64_t, int64_t) {}, warp_cnt);
        if (threadIdx.x == 0) counts[world + s] = (int32_t)c;
    }
    if (threadIdx.x == 0) counts[2 * world] = (int32_t)n_loc;
}

}  // namespace

cudaError_t launch_affinity_plan(const int64_t *idx, const uint8_t *hit, int64_t n, const PlanArgs &a, int32_t *assign,
                                 double *load, int64_t *scratch, int64_t *loc, int64_t *idx_loc, uint8_t *hit_loc,
                                 int64_t *send_order, int32_t *counts, cudaStream_t st) {
    affinity_plan_kernel<<<1, kPlanThreads, 0, st>>>(idx, hit, n, a, assign, load, scratch, loc, idx_loc, hit_loc,
                                                     send_order, counts);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace ac
