// F1: segmentation on the GPU (partition.hpp:58-307, pipeline.hpp:131-138).
//
// partition_mesh (partition.hpp:84-159)
//   seeds: the first is mt19937_64(seed)() mod n (host, libstdc++); every
//   further seed is the lowest-id vertex farthest (in hops) from all seeds so
//   far, unreachable first (:89-106).  The multi-source distance is kept
//   incrementally: each round runs a BFS from the newest seed only and lowers
//   dist[] where it improves (a vertex whose distance does not improve cannot
//   improve its neighbours, so the BFS stops there) -- the same distances as
//   the reference's BFS from all seeds.  seed_bfs_kernel: one CTA, level-
//   synchronous, frontier queues in global memory; seed_argmax_kernel: all
//   SMs, (distance, -id) packed in one 64-bit key, atomicMax.
//   growth (:108-157): one warp replays the reference loop exactly: the part
//   with the smallest size (lowest id on ties) among those with a frontier and
//   below cap = int(ceil(n/k) * 1.1) -- any frontier once all are capped --
//   takes the first unassigned neighbour of its frontier's front vertex; a
//   front vertex without one is popped.  Frontiers are linked lists through
//   next[]; a per-vertex cursor skips neighbours already known to be assigned
//   (assignments never revert, so the first unassigned neighbour is at or
//   after it); 32 neighbours are tested per ballot.
// expand_overlaps (:205-253): one CTA per part; BFS rings from the part over
//   a per-part membership bitmap (atomicOr dedupes a ring like the reference's
//   member[] marks); a last ring larger than the room left keeps its smallest
//   ids (found by bisection on the id); an exhausted component is padded with
//   the smallest unused ids; the sorted member list is the bitmap's set bits
//   in ascending order (build_submesh sorts, :170).
// order_submeshes (:258-307): owners per vertex (count, scan, fill) -> the
//   submesh adjacency as a k x k bitmap (pairs sharing a vertex) -> BFS from
//   mt19937_64(seed)() mod k, neighbours in ascending id, restarts at the
//   smallest unvisited id (one thread: k is small).
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <random>

#include "common.cuh"
#include "segment.h"

namespace smg {

namespace {

constexpr int kSeedThreads = 1024;

// BFS from seeds[r] (round r), lowering dist[] where it improves.  seeds[r]
// for r >= 1 comes from the previous round's argmax key.
__global__ void __launch_bounds__(kSeedThreads) seed_bfs_kernel(const int32_t* __restrict__ offs,
                                                                 const int32_t* __restrict__ cols, int32_t* dist,
                                                                 int32_t* qa, int32_t* qb,
                                                                 const unsigned long long* keys, int32_t* seeds,
                                                                 int r) {
    __shared__ int qn, qn_next;
    if (threadIdx.x == 0) {
        int s = seeds[0];
        if (r > 0) s = (int)(0xFFFFFFFFu - (unsigned)(keys[r - 1] & 0xFFFFFFFFull));
        seeds[r] = s;
        dist[s] = 0;
        qa[0] = s;
        qn = 1;
    }
    __syncthreads();
    int d = 0;
    while (qn > 0) {
        if (threadIdx.x == 0) qn_next = 0;
        __syncthreads();
        const int m = qn;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const int v = qa[i];
            const int e1 = offs[v + 1];
            for (int j = offs[v]; j < e1; ++j) {
                const int w = cols[j];
                if (dist[w] > d + 1) {
                    const int old = atomicMin(&dist[w], d + 1);
                    if (old > d + 1) qb[atomicAdd(&qn_next, 1)] = w;
                }
            }
        }
        __syncthreads();
        int32_t* t = qa;
        qa = qb;
        qb = t;
        if (threadIdx.x == 0) qn = qn_next;
        ++d;
        __syncthreads();
    }
}

// farthest vertex, lowest id on ties: max of (dist << 32 | ~id)
__global__ void seed_argmax_kernel(const int32_t* __restrict__ dist, int n, unsigned long long* key) {
    unsigned long long best = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const unsigned long long k = ((unsigned long long)(unsigned)dist[v] << 32) | (0xFFFFFFFFu - (unsigned)v);
        best = k > best ? k : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(key, best);
}

// The growth loop on one warp (partition.hpp:108-157).  status: 0 ok, 1 no
// part can grow (the reference's "partition failed" InvalidArgument).
__global__ void grow_kernel(const int32_t* __restrict__ offs, const int32_t* __restrict__ cols, int n, int k,
                            int cap, const int32_t* seeds, int32_t* assign, int32_t* next, int32_t* cursor,
                            int* status) {
    extern __shared__ int sm[];
    int* head = sm;
    int* tail = sm + k;
    int* size = sm + 2 * k;
    const int lane = threadIdx.x;
    for (int p = lane; p < k; p += 32) {
        const int s = seeds[p];
        head[p] = tail[p] = s;
        size[p] = 1;
        assign[s] = p;
        next[s] = -1;
    }
    __syncwarp();
    int assigned = k;
    auto pick = [&](bool respect_cap) {
        unsigned long long best = ~0ull;
        for (int p = lane; p < k; p += 32) {
            if (head[p] < 0) continue;
            if (respect_cap && size[p] >= cap) continue;
            const unsigned long long key = ((unsigned long long)(unsigned)size[p] << 32) | (unsigned)p;
            best = key < best ? key : best;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
            best = x < best ? x : best;
        }
        return best == ~0ull ? -1 : (int)(best & 0xFFFFFFFFull);
    };
    while (assigned < n) {
        int p = pick(true);
        if (p < 0) p = pick(false);  // capped everywhere: coverage wins
        if (p < 0) {
            if (lane == 0) *status = 1;
            return;
        }
        bool grew = false;
        while (!grew) {
            const int v = head[p];
            if (v < 0) break;
            const int o0 = offs[v], o1 = offs[v + 1];
            int base = o0 + __ldcg(cursor + v);
            while (base < o1) {
                const int j = base + lane;
                int w = -1;
                bool fr = false;
                if (j < o1) {
                    w = cols[j];
                    fr = __ldcg(assign + w) < 0;
                }
                const unsigned m = __ballot_sync(0xffffffffu, fr);
                if (m) {
                    const int f = __ffs(m) - 1;
                    w = __shfl_sync(0xffffffffu, w, f);
                    if (lane == 0) {
                        assign[w] = p;
                        next[w] = -1;
                        next[tail[p]] = w;
                        tail[p] = w;
                        size[p] += 1;
                        cursor[v] = base + f + 1 - o0;
                    }
                    grew = true;
                    break;
                }
                base += 32;
            }
            if (!grew && lane == 0) {  // v has no unassigned neighbour left: pop it
                cursor[v] = o1 - o0;
                const int nx = __ldcg(next + v);
                head[p] = nx;
                if (nx < 0) tail[p] = -1;
            }
            __syncwarp();
        }
        if (grew) ++assigned;
    }
}

// The same loop, round-parallel and exact.  While no part fails or reaches
// the cap, the serial loop picks the parts of the current minimum size in
// ascending id, each growing by one (after p grows to s+1, every remaining
// size-s part still precedes it): a "round".  All parts of a round propose
// their next vertex at once against the assignment at the round's start
// (front vertices without an unassigned neighbour are popped -- that stays
// true); then the proposals are taken in id order.  A proposal is exactly the
// serial choice unless an earlier part of the round took the same vertex
// (claim[w] = lowest proposer, atomicMin): from the first such collision on,
// the parts are replayed one by one by warp 0 (the rescan sees the earlier
// parts' assignments), which is the serial loop itself.  Rounds of one or two
// parts run serially outright.
constexpr int kGrowWarps = 32;

__global__ void __launch_bounds__(kGrowWarps * 32) grow_rounds_kernel(const int32_t* __restrict__ offs,
                                                                      const int32_t* __restrict__ cols, int n, int k,
                                                                      int cap, const int32_t* seeds, int32_t* assign,
                                                                      int32_t* next, int32_t* cursor, int32_t* claim,
                                                                      int* status) {
    extern __shared__ int sm[];
    int* head = sm;
    int* tail = sm + k;
    int* size = sm + 2 * k;
    int* R = sm + 3 * k;      // this round's parts, ascending id
    int* prop = sm + 4 * k;   // proposed vertex (-1: frontier exhausted)
    int* pcur = sm + 5 * k;   // cursor value after the proposal
    int* pv = sm + 6 * k;     // front vertex the proposal came from
    __shared__ int nR, smin_cap, smin_any, assigned_s, first_conflict, err;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int p = tid; p < k; p += blockDim.x) {
        const int s = seeds[p];
        head[p] = tail[p] = s;
        size[p] = 1;
        assign[s] = p;
        next[s] = -1;
    }
    if (tid == 0) {
        assigned_s = k;
        err = 0;
    }
    __syncthreads();
    // one-warp replay of a pick of part p (the serial loop's body); returns grew
    auto serial_pick = [&](int p) -> bool {
        bool grew = false;
        while (!grew) {
            const int v = head[p];
            if (v < 0) break;
            const int o0 = offs[v], o1 = offs[v + 1];
            int base = o0 + __ldcg(cursor + v);
            while (base < o1) {
                const int j = base + lane;
                int w = -1;
                bool fr = false;
                if (j < o1) {
                    w = cols[j];
                    fr = __ldcg(assign + w) < 0;
                }
                const unsigned m = __ballot_sync(0xffffffffu, fr);
                if (m) {
                    const int f = __ffs(m) - 1;
                    w = __shfl_sync(0xffffffffu, w, f);
                    if (lane == 0) {
                        assign[w] = p;
                        next[w] = -1;
                        next[tail[p]] = w;
                        tail[p] = w;
                        size[p] += 1;
                        cursor[v] = base + f + 1 - o0;
                    }
                    grew = true;
                    break;
                }
                base += 32;
            }
            if (!grew && lane == 0) {
                cursor[v] = o1 - o0;
                const int nx = __ldcg(next + v);
                head[p] = nx;
                if (nx < 0) tail[p] = -1;
            }
            __syncwarp();
        }
        return grew;
    };
    while (true) {
        // ---- the round: parts of the minimum size among those with a frontier
        // below cap (or, once every such part is capped, among all with one)
        if (tid == 0) {
            smin_cap = INT_MAX;
            smin_any = INT_MAX;
            nR = 0;
            first_conflict = INT_MAX;
        }
        __syncthreads();
        if (assigned_s >= n) break;
        for (int p = tid; p < k; p += blockDim.x)
            if (head[p] >= 0) {
                atomicMin(&smin_any, size[p]);
                if (size[p] < cap) atomicMin(&smin_cap, size[p]);
            }
        __syncthreads();
        const bool capmode = smin_cap != INT_MAX;
        const int smin = capmode ? smin_cap : smin_any;
        if (smin == INT_MAX) {
            if (tid == 0) *status = 1;
            return;
        }
        // compaction in id order (warp-level ballots, warps in order)
        if (warp == 0) {
            int cnt = 0;
            for (int p0 = 0; p0 < k; p0 += 32) {
                const int p = p0 + lane;
                const bool in = p < k && head[p] >= 0 && size[p] == smin && (!capmode || size[p] < cap);
                const unsigned m = __ballot_sync(0xffffffffu, in);
                if (in) R[cnt + __popc(m & ((1u << lane) - 1))] = p;
                cnt += __popc(m);
            }
            if (lane == 0) nR = cnt;
        }
        __syncthreads();
        const int nr = nR;
        if (nr <= 2) {
            if (warp == 0) {
                int grown = 0;
                for (int i = 0; i < nr; ++i) grown += serial_pick(R[i]) ? 1 : 0;
                if (lane == 0) assigned_s += grown;
            }
            __syncthreads();
            continue;
        }
        // ---- proposals, one warp per part (scans read the round-start assignment)
        for (int i = warp; i < nr; i += kGrowWarps) {
            const int p = R[i];
            int w = -1, cur = 0, vv = -1;
            while (true) {
                const int v = head[p];
                if (v < 0) break;
                const int o0 = offs[v], o1 = offs[v + 1];
                int base = o0 + __ldcg(cursor + v);
                bool found = false;
                while (base < o1) {
                    const int j = base + lane;
                    int x = -1;
                    bool fr = false;
                    if (j < o1) {
                        x = cols[j];
                        fr = __ldcg(assign + x) < 0;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, fr);
                    if (m) {
                        const int f = __ffs(m) - 1;
                        w = __shfl_sync(0xffffffffu, x, f);
                        cur = base + f + 1 - o0;
                        vv = v;
                        found = true;
                        break;
                    }
                    base += 32;
                }
                if (found) break;
                if (lane == 0) {  // exhausted at the round start: exhausted for good
                    cursor[v] = o1 - o0;
                    const int nx = __ldcg(next + v);
                    head[p] = nx;
                    if (nx < 0) tail[p] = -1;
                }
                __syncwarp();
            }
            if (lane == 0) {
                prop[i] = w;
                pcur[i] = cur;
                pv[i] = vv;
                if (w >= 0) atomicMin(claim + w, i);
            }
        }
        __syncthreads();
        // ---- first collision in id order
        for (int i = tid; i < nr; i += blockDim.x)
            if (prop[i] >= 0 && __ldcg(claim + prop[i]) != i) atomicMin(&first_conflict, i);
        __syncthreads();
        const int cfl = first_conflict;
        // the collision-free prefix commits in parallel
        int grown = 0;
        for (int i = tid; i < min(nr, cfl); i += blockDim.x) {
            const int p = R[i], w = prop[i];
            if (w < 0) continue;
            assign[w] = p;
            next[w] = -1;
            next[tail[p]] = w;
            tail[p] = w;
            size[p] += 1;
            cursor[pv[i]] = pcur[i];
            ++grown;
        }
        grown = __reduce_add_sync(0xffffffffu, grown);
        if (lane == 0 && grown) atomicAdd(&assigned_s, grown);
        __syncthreads();
        // from the collision on: the serial loop (a proposal still stands when
        // no earlier part claimed its vertex and it is still free)
        if (cfl < nr && warp == 0) {
            int g2 = 0;
            for (int i = cfl; i < nr; ++i) {
                const int p = R[i], w = prop[i];
                if (w < 0) continue;  // frontier exhausted: this pick fails
                const bool ok = (__ldcg(claim + w) == i) && (__ldcg(assign + w) < 0);
                if (ok) {
                    if (lane == 0) {
                        assign[w] = p;
                        next[w] = -1;
                        next[tail[p]] = w;
                        tail[p] = w;
                        size[p] += 1;
                        cursor[pv[i]] = pcur[i];
                    }
                    __syncwarp();
                    ++g2;
                } else {
                    g2 += serial_pick(p) ? 1 : 0;
                }
            }
            if (lane == 0) assigned_s += g2;
        }
        __syncthreads();
        for (int i = tid; i < nr; i += blockDim.x)
            if (prop[i] >= 0) claim[prop[i]] = INT_MAX;
        __syncthreads();
    }
}

// ------------------------------------------------------------------ expand_overlaps

constexpr int kExpThreads = 512;

// Block-wide exclusive scan of one int per thread (returns the prefix, total in *tot).
__device__ int block_exclusive_scan(int v, int* scratch /* >= 32 */, int* tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) scratch[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < nw ? scratch[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) scratch[lane] = s;
    }
    __syncthreads();
    const int before = (wid > 0 ? scratch[wid - 1] : 0) + x - v;
    *tot = scratch[nw - 1];
    __syncthreads();
    return before;
}

struct ExpandParams {
    const int32_t* offs;
    const int32_t* cols;
    int n, words, target;
    const int32_t* poffs;  // members of each raw part (CSR by part)
    const int32_t* plist;
    uint32_t* bitmaps;     // k x words, zeroed
    int32_t* ring;         // k x 2 x ring_cap
    int64_t ring_cap;
    int32_t* members;      // k x target (sorted per row)
};

__global__ void __launch_bounds__(kExpThreads) expand_kernel(ExpandParams p) {
    __shared__ int scratch[32];
    __shared__ int nq, cnt_below;
    const int part = blockIdx.x;
    uint32_t* M = p.bitmaps + (int64_t)part * p.words;
    int32_t* ra = p.ring + (int64_t)part * 2 * p.ring_cap;
    int32_t* rb = ra + p.ring_cap;
    const int b0 = p.poffs[part], b1 = p.poffs[part + 1];
    int rn = b1 - b0;
    for (int i = threadIdx.x; i < rn; i += blockDim.x) {
        const int v = p.plist[b0 + i];
        atomicOr(&M[v >> 5], 1u << (v & 31));
        ra[i] = v;
    }
    int count = rn;
    __syncthreads();
    while (count < p.target) {
        if (threadIdx.x == 0) nq = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < rn; i += blockDim.x) {
            const int v = ra[i];
            const int e1 = p.offs[v + 1];
            for (int j = p.offs[v]; j < e1; ++j) {
                const int w = p.cols[j];
                const uint32_t bit = 1u << (w & 31);
                if (M[w >> 5] & bit) continue;
                const uint32_t old = atomicOr(&M[w >> 5], bit);
                if (!(old & bit)) rb[atomicAdd(&nq, 1)] = w;
            }
        }
        __syncthreads();
        const int m = nq;
        if (m == 0) break;  // component exhausted
        const int room = p.target - count;
        if (m > room) {
            // keep the room smallest ids: bisect for the largest t with
            // #{w < t} <= room ... the room-th smallest id is the t with #{w <= t} == room
            int lo = 0, hi = p.n - 1;  // answer in [lo, hi]
            while (lo < hi) {
                const int mid = lo + (hi - lo) / 2;
                if (threadIdx.x == 0) cnt_below = 0;
                __syncthreads();
                int c = 0;
                for (int i = threadIdx.x; i < m; i += blockDim.x) c += rb[i] <= mid;
                c = __reduce_add_sync(0xffffffffu, c);
                if ((threadIdx.x & 31) == 0) atomicAdd(&cnt_below, c);
                __syncthreads();
                if (cnt_below >= room) hi = mid;
                else lo = mid + 1;
                __syncthreads();
            }
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int w = rb[i];
                if (w > lo) atomicAnd(&M[w >> 5], ~(1u << (w & 31)));  // trimmed: not a member
            }
            count = p.target;
            __syncthreads();
            break;
        }
        count += m;
        int32_t* t = ra;
        ra = rb;
        rb = t;
        rn = m;
        __syncthreads();
    }
    __syncthreads();
    // words per thread, in order
    const int per = (p.words + blockDim.x - 1) / blockDim.x;
    const int w0 = threadIdx.x * per, w1 = min(p.words, w0 + per);
    auto valid = [&](int wd) {  // bits of word wd that are vertices
        const int lo = wd * 32;
        return (p.n - lo >= 32) ? 0xFFFFFFFFu : ((1u << (p.n - lo)) - 1u);
    };
    if (count < p.target) {
        // disconnected remainder: the smallest unused ids
        int z = 0;
        for (int wd = w0; wd < w1; ++wd) z += __popc(~M[wd] & valid(wd));
        int tot;
        int before = block_exclusive_scan(z, scratch, &tot);
        const int need = p.target - count;
        for (int wd = w0; wd < w1 && before < need; ++wd) {
            uint32_t free = ~M[wd] & valid(wd);
            while (free && before < need) {
                const int b = __ffs(free) - 1;
                free &= free - 1;
                M[wd] |= 1u << b;
                ++before;
            }
        }
        __syncthreads();
    }
    int c = 0;
    for (int wd = w0; wd < w1; ++wd) c += __popc(M[wd]);
    int tot;
    int pos = block_exclusive_scan(c, scratch, &tot);
    int32_t* out = p.members + (int64_t)part * p.target;
    for (int wd = w0; wd < w1; ++wd) {
        uint32_t bits = M[wd];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            if (pos < p.target) out[pos] = wd * 32 + b;
            ++pos;
        }
    }
}

__global__ void part_count_kernel(const int32_t* assign, int n, int32_t* cnt) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) atomicAdd(&cnt[assign[v]], 1);
}

__global__ void part_fill_kernel(const int32_t* assign, int n, const int32_t* offs, int32_t* fill, int32_t* list) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int p = assign[v];
        list[offs[p] + atomicAdd(&fill[p], 1)] = v;
    }
}

__global__ void max_degree_kernel(const int32_t* offs, int n, int* out) {
    int m = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) m = max(m, offs[v + 1] - offs[v]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ------------------------------------------------------------------ order_submeshes

__global__ void owner_count_kernel(const int32_t* members, int64_t total, int32_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[members[i]], 1);
}

__global__ void owner_fill_kernel(const int32_t* members, int64_t total, int n_d, const int32_t* offs, int32_t* fill,
                                  int32_t* owners) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int g = members[i];
        owners[offs[g] + atomicAdd(&fill[g], 1)] = (int)(i / n_d);
    }
}

// every pair of submeshes sharing a vertex is adjacent (partition.hpp:270-275)
__global__ void owner_pairs_kernel(const int32_t* offs, const int32_t* owners, int n, uint32_t* adj, int kw) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
        const int a0 = offs[g], a1 = offs[g + 1];
        for (int a = a0; a < a1; ++a)
            for (int b = a + 1; b < a1; ++b) {
                const int s = owners[a], t = owners[b];
                if (s == t) continue;
                atomicOr(&adj[(int64_t)s * kw + (t >> 5)], 1u << (t & 31));
                atomicOr(&adj[(int64_t)t * kw + (s >> 5)], 1u << (s & 31));
            }
    }
}

// BFS over the submesh graph (partition.hpp:283-306), one thread
__global__ void order_bfs_kernel(const uint32_t* adj, int k, int kw, int initial, int32_t* visited, int32_t* queue) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int qh = 0, qt = 0, nseq = 0, nxt = 0;
    auto visit = [&](int s) {
        visited[s] = 1;
        queue[qt++] = s;  // the queue in visit order is the sequence
        ++nseq;
    };
    visit(initial);
    while (nseq < k) {
        if (qh == qt) {
            while (visited[nxt]) ++nxt;
            visit(nxt);
            continue;
        }
        const int s = queue[qh++];
        const uint32_t* row = adj + (int64_t)s * kw;
        for (int w = 0; w < kw; ++w) {
            uint32_t bits = row[w];
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                const int t = w * 32 + b;
                if (!visited[t]) visit(t);
            }
        }
    }
}

int grid_for(int64_t n, int threads) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)sms * 8));
}

void exclusive_scan(const int32_t* in, int32_t* out, int n, cudaStream_t st) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st);
    DBuf<char> tmp;
    tmp.alloc(bytes, st);
    cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, st);
}

}  // namespace

void partition_mesh_dev(const GraphDev& g, int k, uint64_t seed, int32_t* assignment, cudaStream_t st) {
    const int n = g.n;
    require(k >= 1 && k <= n / 4, "part count k must satisfy 1 <= k <= n/4");
    std::mt19937_64 rng(seed);
    const int32_t s0 = (int32_t)(rng() % (uint64_t)n);
    DBuf<int32_t> dist, qa, qb, seeds, next, cursor;
    DBuf<unsigned long long> keys;
    DBuf<int> status;
    dist.alloc(n, st);
    qa.alloc(n, st);
    qb.alloc(n, st);
    seeds.alloc(k, st);
    keys.alloc(std::max(k, 1), st);
    keys.zero();
    SMG_CUDA(cudaMemsetAsync(dist.get(), 0x7F, sizeof(int32_t) * n, st));  // 0x7F7F7F7F > any hop count
    SMG_CUDA(cudaMemcpyAsync(seeds.get(), &s0, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    const int ag = grid_for(n, 256);
    for (int r = 0; r + 1 < k; ++r) {
        ::smg::count_launch(), seed_bfs_kernel<<<1, kSeedThreads, 0, st>>>(g.offs, g.cols, dist.get(), qa.get(), qb.get(),
                                                                          keys.get(), seeds.get(), r);
        ::smg::count_launch(), seed_argmax_kernel<<<ag, 256, 0, st>>>(dist.get(), n, keys.get() + r);
    }
    if (k > 1) {
        // the last seed from the last argmax (the BFS kernel's prologue does the decode)
        unsigned long long key = 0;
        SMG_CUDA(cudaMemcpyAsync(&key, keys.get() + (k - 2), sizeof(key), cudaMemcpyDeviceToHost, st));
        SMG_CUDA(cudaStreamSynchronize(st));
        const int32_t s = (int32_t)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull));
        SMG_CUDA(cudaMemcpyAsync(seeds.get() + (k - 1), &s, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    }
    next.alloc(n, st);
    cursor.alloc(n, st);
    cursor.zero();
    status.alloc(1, st);
    status.zero();
    SMG_CUDA(cudaMemsetAsync(assignment, 0xFF, sizeof(int32_t) * n, st));  // -1
    const int cap = (int)(std::ceil((double)n / k) * 1.1);
    if (std::getenv("SMG_GROW_SERIAL") || 7 * k * (int)sizeof(int) > 200 * 1024) {
        const int smem = 3 * k * (int)sizeof(int);
        ensure_smem((const void*)grow_kernel, smem);
        ::smg::count_launch(), grow_kernel<<<1, 32, smem, st>>>(g.offs, g.cols, n, k, cap, seeds.get(), assignment,
                                                                next.get(), cursor.get(), status.get());
    } else {
        DBuf<int32_t> claim;
        claim.alloc(n, st);
        SMG_CUDA(cudaMemsetAsync(claim.get(), 0x7F, sizeof(int32_t) * n, st));  // 0x7F7F7F7F > any round index
        const int smem = 7 * k * (int)sizeof(int);
        ensure_smem((const void*)grow_rounds_kernel, smem);
        ::smg::count_launch(), grow_rounds_kernel<<<1, kGrowWarps * 32, smem, st>>>(
            g.offs, g.cols, n, k, cap, seeds.get(), assignment, next.get(), cursor.get(), claim.get(), status.get());
    }
    SMG_CUDA(cudaGetLastError());
    int h = 0;
    SMG_CUDA(cudaMemcpyAsync(&h, status.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    if (h)
        fail(2, "partition failed: k is incompatible with the mesh connectivity "
                "(a component ended up without a seed)");
}

int expand_overlaps_dev(const GraphDev& g, const int32_t* assignment, int k, double growth, DBuf<int32_t>& members,
                        cudaStream_t st) {
    const int n = g.n;
    DBuf<int32_t> cnt, poffs, fill, plist;
    DBuf<int> maxdeg;
    cnt.alloc(k + 1, st);
    cnt.zero();
    poffs.alloc(k + 1, st);
    fill.alloc(k, st);
    fill.zero();
    plist.alloc(n, st);
    maxdeg.alloc(1, st);
    maxdeg.zero();
    const int gr = grid_for(n, 256);
    ::smg::count_launch(), part_count_kernel<<<gr, 256, 0, st>>>(assignment, n, cnt.get());
    ::smg::count_launch(), max_degree_kernel<<<gr, 256, 0, st>>>(g.offs, n, maxdeg.get());
    std::vector<int32_t> sizes = download(cnt.get(), (size_t)k, st);
    int md = download(maxdeg.get(), 1, st)[0];
    for (int p = 0; p < k; ++p) require(sizes[p] > 0, "partition has an empty part");
    const int max_raw = *std::max_element(sizes.begin(), sizes.end());
    require(growth >= 1.0, "overlap growth must be >= 1.0");
    const int target = (int)std::floor(growth * max_raw);
    require(target <= n, "target submesh size exceeds the vertex count");
    exclusive_scan(cnt.get(), poffs.get(), k + 1, st);
    ::smg::count_launch(), part_fill_kernel<<<gr, 256, 0, st>>>(assignment, n, poffs.get(), fill.get(), plist.get());
    ExpandParams p{};
    p.offs = g.offs;
    p.cols = g.cols;
    p.n = n;
    p.words = (n + 31) / 32;
    p.target = target;
    p.poffs = poffs.get();
    p.plist = plist.get();
    // a ring never exceeds the neighbours of the previous (kept) ring, which
    // has at most max(target, largest part) vertices
    p.ring_cap = std::min<int64_t>(n, (int64_t)std::max(target, max_raw) * std::max(md, 1) + 32);
    DBuf<uint32_t> bm;
    DBuf<int32_t> ring;
    bm.alloc((size_t)k * p.words, st);
    bm.zero();
    ring.alloc((size_t)k * 2 * p.ring_cap, st);
    members.alloc((size_t)k * target, st);
    p.bitmaps = bm.get();
    p.ring = ring.get();
    p.members = members.get();
    ::smg::count_launch(), expand_kernel<<<k, kExpThreads, 0, st>>>(p);
    SMG_CUDA(cudaGetLastError());
    SMG_CUDA(cudaStreamSynchronize(st));
    return target;
}

std::vector<int32_t> order_submeshes_dev(const int32_t* members, int k, int n_d, int n, uint64_t seed,
                                         cudaStream_t st) {
    require(k >= 1, "cannot order an empty submesh list");
    require(k <= 16384, "order_submeshes: more than 16384 submeshes");
    const int64_t total = (int64_t)k * n_d;
    DBuf<int32_t> cnt, offs, fill, owners, visited, queue;
    cnt.alloc(n + 1, st);
    cnt.zero();
    offs.alloc(n + 1, st);
    fill.alloc(n, st);
    fill.zero();
    const int gt = grid_for(total, 256), gn = grid_for(n, 256);
    ::smg::count_launch(), owner_count_kernel<<<gt, 256, 0, st>>>(members, total, cnt.get());
    exclusive_scan(cnt.get(), offs.get(), n + 1, st);
    owners.alloc(total, st);
    ::smg::count_launch(), owner_fill_kernel<<<gt, 256, 0, st>>>(members, total, n_d, offs.get(), fill.get(), owners.get());
    const int kw = (k + 31) / 32;
    DBuf<uint32_t> adj;
    adj.alloc((size_t)k * kw, st);
    adj.zero();
    ::smg::count_launch(), owner_pairs_kernel<<<gn, 256, 0, st>>>(offs.get(), owners.get(), n, adj.get(), kw);
    std::mt19937_64 rng(seed);
    const int initial = (int)(rng() % (uint64_t)k);
    visited.alloc(k, st);
    visited.zero();
    queue.alloc(k, st);
    ::smg::count_launch(), order_bfs_kernel<<<1, 32, 0, st>>>(adj.get(), k, kw, initial, visited.get(), queue.get());
    SMG_CUDA(cudaGetLastError());
    return download(queue.get(), (size_t)k, st);
}

void segment_mesh_dev(const GraphDev& g, int k, double growth, uint64_t seed, DeviceSegmentation& out,
                      cudaStream_t st) {
    out.k = k;
    out.assignment.alloc(g.n, st);
    partition_mesh_dev(g, k, seed, out.assignment.get(), st);
    out.n_d = expand_overlaps_dev(g, out.assignment.get(), k, growth, out.members, st);
    out.sequence_h = order_submeshes_dev(out.members.get(), k, out.n_d, g.n, seed, st);
    out.offsets_h.resize(k + 1);
    for (int s = 0; s <= k; ++s) out.offsets_h[s] = s * out.n_d;
    out.offsets.upload(out.offsets_h, st);
}

}  // namespace smg

// ------------------------------------------------------------------ C ABI
#include "../../include/specmesh_gpu.h"
#include "context.h"

namespace {

struct GraphStage {
    smg::GraphDev g;
    smg::DBuf<int32_t> offs, cols;
};

void stage_graph(const smg_mesh* m, GraphStage& s, cudaStream_t st) {
    smg::require(m != nullptr, "mesh view is null");
    smg::require(m->vertex_count >= 0 && m->vertex_count < INT_MAX, "mesh vertex count out of range");
    s.g.n = (int)m->vertex_count;
    if (m->on_device) {
        s.g.offs = m->adj_offsets;
        s.g.cols = m->adj_cols;
        return;
    }
    s.offs.upload(m->adj_offsets, (size_t)s.g.n + 1, st);
    s.cols.upload(m->adj_cols, (size_t)m->adj_offsets[s.g.n], st);
    s.g.offs = s.offs.get();
    s.g.cols = s.cols.get();
}

template <class F>
smg_status seg_guard(smg_context* ctx, F&& f) {
    return static_cast<smg_status>(smg::guarded_call(ctx, std::forward<F>(f)));
}

}  // namespace

extern "C" {

smg_status smg_partition_mesh(smg_context* ctx, const smg_mesh* mesh, int32_t part_count, uint64_t seed,
                              int32_t* assignment) {
    return seg_guard(ctx, [&] {
        smg::require(assignment != nullptr, "assignment output is null");
        const cudaStream_t st = ctx->stream;
        GraphStage gs;
        stage_graph(mesh, gs, st);
        smg::DBuf<int32_t> a;
        a.alloc(gs.g.n, st);
        smg::partition_mesh_dev(gs.g, part_count, seed, a.get(), st);
        SMG_CUDA(cudaMemcpyAsync(assignment, a.get(), sizeof(int32_t) * gs.g.n, cudaMemcpyDefault, st));
        SMG_CUDA(cudaStreamSynchronize(st));
    });
}

smg_status smg_expand_overlaps(smg_context* ctx, const smg_mesh* mesh, const int32_t* assignment, int32_t part_count,
                               double growth, int32_t* members, int64_t members_capacity, int32_t* block_size) {
    return seg_guard(ctx, [&] {
        smg::require(assignment != nullptr && block_size != nullptr, "assignment / block size pointer is null");
        smg::require(part_count >= 1, "part count must be positive");
        const cudaStream_t st = ctx->stream;
        GraphStage gs;
        stage_graph(mesh, gs, st);
        smg::DBuf<int32_t> a, mem;
        a.upload(assignment, gs.g.n, st);
        std::vector<int32_t> ah(assignment, assignment + gs.g.n);
        for (int32_t v : ah) smg::require(v >= 0 && v < part_count, "assignment entry outside [0, part_count)");
        const int nd = smg::expand_overlaps_dev(gs.g, a.get(), part_count, growth, mem, st);
        *block_size = nd;
        smg::require(members != nullptr && members_capacity >= (int64_t)part_count * nd,
                     "members capacity too small: need part_count * n_d = " +
                         std::to_string((int64_t)part_count * nd));
        SMG_CUDA(cudaMemcpyAsync(members, mem.get(), sizeof(int32_t) * (size_t)part_count * nd, cudaMemcpyDefault, st));
        SMG_CUDA(cudaStreamSynchronize(st));
    });
}

smg_status smg_order_submeshes(smg_context* ctx, int32_t submesh_count, const int32_t* member_offsets,
                               const int32_t* members, uint64_t seed, int32_t* sequence) {
    return seg_guard(ctx, [&] {
        smg::require(submesh_count >= 1, "cannot order an empty submesh list");
        smg::require(member_offsets && members && sequence, "segmentation arrays are null");
        const cudaStream_t st = ctx->stream;
        // ragged lists are padded to the longest with its own last entry
        // (a repeated owner adds no new pair)
        int nd = 0, maxv = -1;
        for (int s = 0; s < submesh_count; ++s) {
            nd = std::max(nd, member_offsets[s + 1] - member_offsets[s]);
            smg::require(member_offsets[s + 1] > member_offsets[s], "submesh has no vertices");
        }
        std::vector<int32_t> flat((size_t)submesh_count * nd);
        for (int s = 0; s < submesh_count; ++s) {
            const int b = member_offsets[s], e = member_offsets[s + 1];
            for (int i = 0; i < nd; ++i) {
                const int32_t v = members[std::min(b + i, e - 1)];
                smg::require(v >= 0, "negative vertex id");
                flat[(size_t)s * nd + i] = v;
                maxv = std::max(maxv, v);
            }
        }
        smg::DBuf<int32_t> mem;
        mem.upload(flat, st);
        std::vector<int32_t> seq = smg::order_submeshes_dev(mem.get(), submesh_count, nd, maxv + 1, seed, st);
        std::copy(seq.begin(), seq.end(), sequence);
    });
}

smg_status smg_segment_mesh(smg_context* ctx, const smg_mesh* mesh, int32_t part_count, double growth, uint64_t seed,
                            int32_t* assignment, int32_t* members, int64_t members_capacity, int32_t* block_size,
                            int32_t* sequence) {
    return seg_guard(ctx, [&] {
        smg::require(block_size != nullptr && sequence != nullptr, "block size / sequence pointer is null");
        const cudaStream_t st = ctx->stream;
        GraphStage gs;
        stage_graph(mesh, gs, st);
        smg::DeviceSegmentation seg;
        smg::segment_mesh_dev(gs.g, part_count, growth, seed, seg, st);
        *block_size = seg.n_d;
        smg::require(members != nullptr && members_capacity >= (int64_t)part_count * seg.n_d,
                     "members capacity too small: need part_count * n_d = " +
                         std::to_string((int64_t)part_count * seg.n_d));
        if (assignment)
            SMG_CUDA(cudaMemcpyAsync(assignment, seg.assignment.get(), sizeof(int32_t) * gs.g.n, cudaMemcpyDefault, st));
        SMG_CUDA(cudaMemcpyAsync(members, seg.members.get(), sizeof(int32_t) * (size_t)part_count * seg.n_d,
                                 cudaMemcpyDefault, st));
        SMG_CUDA(cudaStreamSynchronize(st));
        std::copy(seg.sequence_h.begin(), seg.sequence_h.end(), sequence);
    });
}

}  // extern "C"
