// sem.cu -- a2: semantic retrieval S_sem as an EXACT GPU scan.
//
// The paper retrieves the top-N MIPS neighbours of the target hidden state
// over the LM-head rows with HNSW (App. A.3). HNSW
// approximates the exact answer; on a B200 the exact scan q . E^T over all
// 128k rows is one HBM pass (~1 GB, ~160 us), so we compute the exact answer
// (reading C2 in DESIGN.md) and select the top-N by (score desc, id asc).
//
// Kernels:
//   sem_scan_kernel     s64[v] = sum_c q[c] E[v][c] in fp64 (bf16 x fp32 products
//                       are exact in fp64), one warp per 16-row chunk, 16-byte
//                       streaming loads, q held per lane from a lane-interleaved
//                       fp64 copy in shared memory.
//                       The scan also histograms the top 12 bits of the
//                       order-preserving fp32 key of every score.
//   topn_cand_kernel    grid-wide radix select over the composite key
//                       (float_key(s), double_key(s), ~id). Pass 0 reuses the
//                       scan's histogram, so in the common case no grid-wide
//                       sync runs: every CTA finds the boundary bin b and emits
//                       all scores in bins >= b -- a candidate SUPERSET of the
//                       top-N of at most `cap` elements, carrying exact keys.
//                       Further passes (soft_grid_sync) run only if that superset
//                       would not fit. The exact top-N, its order where the
//                       formation needs it, and the cap are resolved in the
//                       union kernel (union.cu) on those exact keys.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"


namespace es {

// ---------------------------------------------------------------- scan
// Block: kScanWarps warps; each warp owns a contiguous row range and walks it
// in chunks of 16 rows. Per chunk and per 256-column slab (bf16; 128 for
// fp32) each lane loads one 16-byte piece of each of the 16 rows.
template <int DT>  // element type of E: 0 bf16, 1 fp32
__global__ void __launch_bounds__(kScanWarps * 32, 1)
sem_scan_kernel(const void* __restrict__ E, int64_t n_rows, int d,
                const void* __restrict__ q, int q_dtype, uint32_t* __restrict__ hist12,
                double* __restrict__ s64, uint32_t* __restrict__ key32, uint32_t* __restrict__ zero_w, int n_zero_w,
                int* __restrict__ zero_c) {
    // zero the candidate selection's scratch for the next kernel (saves two memsets)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_zero_w; i += gridDim.x * blockDim.x) zero_w[i] = 0;
    if (zero_c && blockIdx.x == 0 && threadIdx.x == 0) *zero_c = 0;
    constexpr int ELEMS = DT == 0 ? 8 : 4;           // elements per 16 bytes
    constexpr int SLAB = 32 * ELEMS;                  // columns per slab
    extern __shared__ double q_sm[];                  // [n_slabs][ELEMS][32]
    __shared__ uint32_t hist_sm[kHistBins];           // top-12-bit histogram of key32
    const int n_slabs = (d + SLAB - 1) / SLAB;
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist_sm[i] = 0;
    // stage q as fp64 in the lane-interleaved layout (exact: q is bf16/fp32)
    for (int i = threadIdx.x; i < n_slabs * SLAB; i += blockDim.x) {
        int s = i / SLAB, within = i % SLAB, lane = within / ELEMS, j = within % ELEMS;
        int c = s * SLAB + within;
        double v = 0.0;
        if (c < d) v = q_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)q)[c])
                                    : (double)((const float*)q)[c];
        // bf16 E: q is pre-scaled by 2^896 (exact; |q| < 2^128 stays finite) so
        // that each E element can enter as the "raw" double whose fields are the
        // bf16 fields in place (value e * 2^-896, exact, no conversion unit):
        // the product q*e, hence every fma, is bit-identical to the unscaled one
        if (DT == 0) v *= 0x1p896;
        q_sm[(s * ELEMS + j) * 32 + lane] = v;
    }
    __syncthreads();

    const int lane = lane_id();
    const int64_t gw = (int64_t)blockIdx.x * kScanWarps + warp_id();
    const int64_t nw = (int64_t)gridDim.x * kScanWarps;
    const int64_t r0 = n_rows * gw / nw, r1 = n_rows * (gw + 1) / nw;
    const size_t row_bytes = (size_t)d * (DT == 0 ? 2 : 4);

    for (int64_t base = r0; base < r1; base += 16) {
        double acc[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[r] = 0.0;
        for (int s = 0; s < n_slabs; ++s) {
            const int c0 = s * SLAB + lane * ELEMS;
            const bool col_ok = c0 < d;
            uint4 u[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                int64_t row = base + r;
                if (col_ok && row < r1)
                    u[r] = ld_stream((const char*)E + row * row_bytes + (size_t)c0 * (DT == 0 ? 2 : 4));
                else
                    u[r] = make_uint4(0, 0, 0, 0);
            }
            double qv[ELEMS];
#pragma unroll
            for (int j = 0; j < ELEMS; ++j) qv[j] = q_sm[(s * ELEMS + j) * 32 + lane];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if constexpr (DT == 0) {
                    const uint32_t w4[4] = {u[r].x, u[r].y, u[r].z, u[r].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        // sign | exp | mant of a bf16 moved to the double's field positions:
                        // arithmetic >> 3 puts exp at [27:20], mant at [19:13]; the mask
                        // keeps the sign at bit 31 (bf16 zero / denormal map exactly too)
                        const uint32_t lo = (uint32_t)((int32_t)(w4[j] << 16) >> 3) & 0x8FFFE000u;
                        const uint32_t hi = (uint32_t)((int32_t)w4[j] >> 3) & 0x8FFFE000u;
                        acc[r] = fma(__hiloint2double((int)lo, 0), qv[2 * j], acc[r]);
                        acc[r] = fma(__hiloint2double((int)hi, 0), qv[2 * j + 1], acc[r]);
                    }
                } else {
                    float f[4] = {__uint_as_float(u[r].x), __uint_as_float(u[r].y),
                                  __uint_as_float(u[r].z), __uint_as_float(u[r].w)};
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[r] = fma((double)f[j], qv[j], acc[r]);
                }
            }
        }
        // reduce-scatter 16 rows over 32 lanes: lane l ends with row (l & 15)
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
            const bool upper = (lane & h) != 0;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                double send = upper ? acc[i] : acc[i + h];
                double keep = upper ? acc[i + h] : acc[i];
                acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
            }
        }
        double tot = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 16);
        int64_t row = base + (lane & 15);
        uint32_t digit = 0xFFFFFFFFu;
        if (lane < 16 && row < r1) {
            const uint32_t k = float_key((float)tot);
            s64[row] = tot;
            key32[row] = k;
            digit = k >> 20;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (digit != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist_sm[digit], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
        if (hist_sm[i]) atomicAdd(&hist12[i], hist_sm[i]);
}

// per-kernel globaltimer stamps of the build (EVOSPEC_TRACE; profiling aid):
// scan CTA b start / end at [2b], [2b + 1]; the candidate kernel's CTA 0 at [2 * 148], [+1]
static long long* s_step_trace = nullptr;
void set_step_trace(long long* p) { s_step_trace = p; }
ES_DEV long long step_gtime() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- scan (TMA ring)
// bf16 E, d % 256 == 0, d <= 4096: the same exact fp64 scores as above, with E
// streamed through shared memory by the bulk-copy engine instead of per-lane
// loads, so that the bytes in flight per SM stay at the ring size (no drain
// between column slabs).
//   CTA: rows [r0, r1) (contiguous, 1/grid of E); stage = 8 consecutive rows
//   (8 * d * 2 bytes, one contiguous cp.async.bulk); a ring of kScanStages.
//   warp 16: producer (one elected thread). Warps 0 .. d/256-1: consumers; warp
//   w owns the 256-column slab [256 w, 256 w + 256) of every row, q for it lives
//   in registers (8 fp64 per lane, pre-scaled by 2^896), and each stage costs
//   it 8 LDS.128 + 64 fp64 FMAs per lane. A reduce-scatter over the lanes
//   leaves one partial per (row, slab); the stage's owner warp (stage % slabs)
//   adds the partials of each row in slab order and writes s64 / key32 / the
//   histogram, then frees the stage (the others free it right after their
//   partials are written).
constexpr int kScanConsumers = 16;
constexpr int kScanRS = 8;          // rows per ring stage (8: one CTA per SM; measured r2: 4 rows x 6 stages
                                    // 240 us, 2 x 12 358 us vs 195 us -- the per-stage work dominates)

ES_DEV uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
ES_DEV void s_mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n));
}
ES_DEV void s_mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
ES_DEV void s_mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
ES_DEV void s_mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(s_u32(b)), "r"(parity) : "memory");
}
ES_DEV void s_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar)), "l"(policy) : "memory");
}

template <int kScanRowsPerStage, int kScanStages>
__global__ void __launch_bounds__((kScanConsumers + 1) * 32, 1)
sem_scan_tma_kernel(const uint16_t* __restrict__ E, int64_t n_rows, int d, const void* __restrict__ q, int q_dtype,
                    uint32_t* __restrict__ hist12, double* __restrict__ s64, uint32_t* __restrict__ key32,
                    int* __restrict__ sched, uint32_t* __restrict__ zero_w, int n_zero_w, int* __restrict__ zero_c,
                    long long* __restrict__ tr) {
    if (tr && threadIdx.x == 0) tr[2 * blockIdx.x] = step_gtime();
    // launched behind static_bits_kernel (PDL): overlaps it, and waits for it before
    // completing (below), so kernels after the scan see the static bitmap
    pdl_trigger();
    // zero the candidate selection's scratch for the next kernel (saves two memsets)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_zero_w; i += gridDim.x * blockDim.x) zero_w[i] = 0;
    if (zero_c && blockIdx.x == 0 && threadIdx.x == 0) *zero_c = 0;
    extern __shared__ __align__(128) unsigned char sc_sm[];
    const size_t row_bytes = (size_t)d * 2;
    const size_t stage_bytes = kScanRowsPerStage * row_bytes;
    unsigned char* ring = sc_sm;                                              // [S][8][d] bf16
    uint32_t* hist_sm = (uint32_t*)(ring + kScanStages * stage_bytes);       // [4096]
    double* red = (double*)(hist_sm + kHistBins);                            // [2S][16][8]
    uint64_t* full = (uint64_t*)(red + 2 * kScanStages * kScanConsumers * kScanRowsPerStage);
    uint64_t* empty = full + kScanStages;
    uint64_t* part_bar = empty + kScanStages;                                // [2S]
    int64_t* srow = (int64_t*)(part_bar + 2 * kScanStages);                  // [S] first row of the slot's stage
    const int warp = warp_id(), lane = lane_id();
    const int n_slab = d / 256;                                              // <= 16
    // stages are groups of 8 consecutive rows handed out by a global counter (sched[0]):
    // an SM that streams faster takes more of them, so the CTAs end together
    const int n_groups = (int)((n_rows + kScanRowsPerStage - 1) / kScanRowsPerStage);
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist_sm[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kScanStages; ++s) {
            s_mbar_init(&full[s], 1);
            s_mbar_init(&empty[s], n_slab);
            s_mbar_init(&part_bar[s], n_slab);
            s_mbar_init(&part_bar[s + kScanStages], n_slab);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kScanConsumers) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            int g = atomicAdd(&sched[0], 1);
            for (int i = 0;; ++i) {
                const int slot = i % kScanStages;
                if (i >= kScanStages) s_mbar_wait(&empty[slot], (uint32_t)((i / kScanStages) - 1) & 1);
                if (g >= n_groups) {   // no stage left: an end marker (a plain arrive completes the phase)
                    srow[slot] = -1;
                    s_mbar_arrive(&full[slot]);
                    break;
                }
                const int g_next = atomicAdd(&sched[0], 1);   // the next claim overlaps this copy
                const int64_t row = (int64_t)g * kScanRowsPerStage;
                const int nr = (int)min((int64_t)kScanRowsPerStage, n_rows - row);
                const uint32_t bytes = (uint32_t)(nr * row_bytes);
                srow[slot] = row;
                s_mbar_expect(&full[slot], bytes);
                s_bulk_g2s(ring + slot * stage_bytes, (const unsigned char*)E + row * row_bytes, bytes, &full[slot], pol);
                g = g_next;
            }
        }
        return;
    }
    if (warp >= n_slab) return;                  // d < 4096: fewer slab warps
    // q for this warp's slab, lane's 8 columns, fp64 pre-scaled by 2^896 (see sem_scan_kernel)
    double qv[8];
    {
        const int c0 = warp * 256 + lane * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const double v = q_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)q)[c0 + j])
                                          : (double)((const float*)q)[c0 + j];
            qv[j] = v * 0x1p896;
        }
    }
    // this lane's 16 bytes of its slab in row 0 of slot 0, as a shared-window address
    const uint32_t my_s = s_u32(ring) + (uint32_t)(warp * 512 + lane * 16);
    for (int i = 0;; ++i) {
        const int slot = i % kScanStages;
        s_mbar_wait(&full[slot], (uint32_t)(i / kScanStages) & 1);
        const int64_t row0 = srow[slot];
        if (row0 < 0) break;
        const int nr = (int)min((int64_t)kScanRowsPerStage, n_rows - row0);
        const uint32_t st = my_s + (uint32_t)(slot * stage_bytes);
        // this warp's slab of the stage into registers, then the slot goes back to
        // the producer at once: the ring refills while the warp computes
        uint4 u[kScanRowsPerStage];
        if (nr == kScanRowsPerStage) {
#pragma unroll
            for (int r = 0; r < kScanRowsPerStage; ++r)
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(u[r].x), "=r"(u[r].y), "=r"(u[r].z), "=r"(u[r].w)
                             : "r"(st + (uint32_t)(r * row_bytes)) : "memory");
        } else {
#pragma unroll
            for (int r = 0; r < kScanRowsPerStage; ++r) {
                u[r] = make_uint4(0, 0, 0, 0);
                if (r < nr)
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(u[r].x), "=r"(u[r].y), "=r"(u[r].z), "=r"(u[r].w)
                                 : "r"(st + (uint32_t)(r * row_bytes)) : "memory");
            }
        }
        // every lane orders its generic-proxy reads of the slot before the async-proxy
        // (bulk copy) refill that the release lets the producer issue
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) s_mbar_arrive(&empty[slot]);
        double acc[kScanRowsPerStage];
#pragma unroll
        for (int r = 0; r < kScanRowsPerStage; ++r) {
            double a_lo = 0.0, a_hi = 0.0;   // two chains of 4 (latency), summed at the end
            const uint32_t w4[4] = {u[r].x, u[r].y, u[r].z, u[r].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // bf16 fields in place in the double's high word (see sem_scan_kernel)
                const uint32_t lo = (uint32_t)((int32_t)(w4[j] << 16) >> 3) & 0x8FFFE000u;
                const uint32_t hi = (uint32_t)((int32_t)w4[j] >> 3) & 0x8FFFE000u;
                a_lo = fma(__hiloint2double((int)lo, 0), qv[2 * j], a_lo);
                a_hi = fma(__hiloint2double((int)hi, 0), qv[2 * j + 1], a_hi);
            }
            acc[r] = a_lo + a_hi;
        }
        // reduce-scatter 8 rows over 32 lanes: lanes (l & 7) == r end with row r's
        // sum over 4 lanes, then two butterflies finish it
#pragma unroll
        for (int h = kScanRowsPerStage / 2; h >= 1; h >>= 1) {
            const bool upper = (lane & h) != 0;
#pragma unroll
            for (int k = 0; k < h; ++k) {
                const double send = upper ? acc[k] : acc[k + h];
                const double keep = upper ? acc[k + h] : acc[k];
                acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
            }
        }
        double part = acc[0];
#pragma unroll
        for (int o = kScanRowsPerStage; o < 32; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        // partials double-buffered over 2S stages: a warp is at most S stages ahead of
        // the owner of stage i (the owner must load stage i + S before the slot of
        // stage i + 2S can refill), so stage i + 2S never overwrites unread partials
        const int pslot = i % (2 * kScanStages);
        double* rd = red + (size_t)pslot * kScanConsumers * kScanRowsPerStage;
        if (lane < kScanRowsPerStage) rd[warp * kScanRowsPerStage + lane] = part;   // lane r holds row r
        __syncwarp();
        if (lane == 0) s_mbar_arrive(&part_bar[pslot]);
        if (warp != i % n_slab) continue;
        // owner: the 16 partials of each row, added in slab order
        s_mbar_wait(&part_bar[pslot], (uint32_t)(i / (2 * kScanStages)) & 1);
        uint32_t digit = 0xFFFFFFFFu;
        if (lane < nr) {
            double tot = 0.0;
            for (int w = 0; w < n_slab; ++w) tot += rd[w * kScanRowsPerStage + lane];
            const int64_t row = row0 + lane;
            const uint32_t kk = float_key((float)tot);
            s64[row] = tot;
            key32[row] = kk;
            digit = kk >> 20;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (digit != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist_sm[digit], (uint32_t)__popc(peers));
        __syncwarp();
    }
    // every slab warp has retired its stages; merge the histogram
    asm volatile("bar.sync 1, %0;" ::"r"(n_slab * 32) : "memory");
    for (int i = threadIdx.x; i < kHistBins; i += n_slab * 32)
        if (hist_sm[i]) atomicAdd(&hist12[i], hist_sm[i]);
    if (tr && threadIdx.x == 0) tr[2 * blockIdx.x + 1] = step_gtime();
    if (threadIdx.x == 0) {
        // the last CTA out resets the stage counter for the next launch (every CTA's
        // claims precede its arrival here)
        __threadfence();
        if (atomicAdd(&sched[1], 1) == (int)gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
            __threadfence();
        }
        pdl_wait();
    }
}

void launch_sem_scan(const void* E, int e_dtype, int64_t n_rows, int d, const void* q, int q_dtype,
                     double* s64, uint32_t* key32, uint32_t* hist12, cudaStream_t st, uint32_t* zero_w,
                     int n_zero_w, int* zero_c, bool hist_zero, int* sched) {
    // hist_zero: hist12 is already zero (the previous build's union kernel cleared it)
    if (!hist_zero) cudaMemsetAsync(hist12, 0, kHistBins * sizeof(uint32_t), st);
    const int elems = e_dtype == 0 ? 8 : 4;
    const int n_slabs = (d + 32 * elems - 1) / (32 * elems);
    const size_t smem = (size_t)n_slabs * 32 * elems * sizeof(double);
    // 8-row stages (64 KB at d = 4096) in a 3-stage ring, one CTA per SM (4- and
    // 2-row stages measured slower: per-stage overhead)
    constexpr int RS = kScanRS, NS = 3;
    auto smem_for = [&](int rs, int ns) {
        return (size_t)ns * rs * d * 2 + kHistBins * 4 + (size_t)2 * ns * kScanConsumers * rs * 8 + 5 * ns * 8;
    };
    // EVOSPEC_SCAN_RING2=1 (test only, tests/test_gpu_scan_ring.py): a 2-stage ring -- every
    // slot is refilled while the slab warps of the stage before it still compute, the
    // tightest reuse of the release / refill ordering; the scores must equal the 3-stage
    // ring's bit for bit (same summation order)
    static const bool ring2 = getenv("EVOSPEC_SCAN_RING2") != nullptr;
    if (e_dtype == 0 && sched && d % 256 == 0 && d <= 256 * kScanConsumers && smem_for(RS, NS) <= 227 * 1024) {
        const size_t sm = smem_for(RS, ring2 ? 2 : NS);
        static thread_local size_t attr = 0, attr2 = 0;
        if (ring2) {
            if (attr2 < sm) {
                cudaFuncSetAttribute(sem_scan_tma_kernel<RS, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                attr2 = sm;
            }
            launch_pdl(sem_scan_tma_kernel<RS, 2>, dim3(kNumSMs), dim3((kScanConsumers + 1) * 32), sm, st,
                       (const uint16_t*)E, n_rows, d, q, q_dtype, hist12, s64, key32, sched, zero_w, n_zero_w,
                       zero_c, s_step_trace);
            return;
        }
        if (attr < sm) {
            cudaFuncSetAttribute(sem_scan_tma_kernel<RS, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            attr = sm;
        }
        launch_pdl(sem_scan_tma_kernel<RS, NS>, dim3(kNumSMs), dim3((kScanConsumers + 1) * 32), sm, st,
                   (const uint16_t*)E, n_rows, d, q, q_dtype, hist12, s64, key32, sched, zero_w, n_zero_w, zero_c,
                   s_step_trace);
    } else if (e_dtype == 0) {
        cudaFuncSetAttribute(sem_scan_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sem_scan_kernel<0><<<kNumSMs, kScanWarps * 32, smem, st>>>(E, n_rows, d, q, q_dtype, hist12, s64, key32,
                                                                    zero_w, n_zero_w, zero_c);
    } else {
        cudaFuncSetAttribute(sem_scan_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sem_scan_kernel<1><<<kNumSMs, kScanWarps * 32, smem, st>>>(E, n_rows, d, q, q_dtype, hist12, s64, key32,
                                                                    zero_w, n_zero_w, zero_c);
    }
}

// ---------------------------------------------------------------- select
struct SelWords { uint32_t w[4]; };

ES_DEV SelWords sel_words(double s, int32_t id) {
    SelWords k;
    k.w[0] = float_key((float)s);
    uint64_t dk = double_key(s);
    k.w[1] = (uint32_t)(dk >> 32);
    k.w[2] = (uint32_t)dk;
    k.w[3] = 0xFFFFFFFFu - (uint32_t)id;   // lower id ranks higher
    return k;
}

struct SelState {
    uint32_t pmask[4], pval[4];
    int remaining;
    int done;
};

ES_DEV bool sel_matches(const SelWords& k, const SelState& st) {
#pragma unroll
    for (int w = 0; w < 4; ++w)
        if ((k.w[w] & st.pmask[w]) != st.pval[w]) return false;
    return true;
}
// composite-prefix >= selected prefix
ES_DEV bool sel_selected(const SelWords& k, const SelState& st) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        uint32_t a = k.w[w] & st.pmask[w];
        if (a != st.pval[w]) return a > st.pval[w];
    }
    return true;
}

// digit schedule: word 0 (fp32 key) 12/10/10 bits -- pass 0 matches the
// scan's 4096-bin histogram; words 1-3: 11/11/10 bits.
ES_DEV void pass_digit(int pass, int& word, int& shift, int& nbits) {
    word = pass / 3;
    const int part = pass % 3;
    if (word == 0) { shift = part == 0 ? 20 : (part == 1 ? 10 : 0); nbits = part == 0 ? 12 : 10; }
    else { shift = part == 0 ? 21 : (part == 1 ? 10 : 0); nbits = part == 2 ? 10 : 11; }
}

// Grid barrier for topn_cand_kernel's rare multi-pass path, without a cooperative
// launch (whose start waits for the whole predecessor grid to drain): every CTA runs
// griddepcontrol.launch_dependents first, so no later kernel of the stream is scheduled
// before all of this grid's CTAs are resident, and waiting CTAs cannot starve the
// others. One counter, never reset: CTA 0 adds 2^31 - (G - 1), the others 1, so the
// top bit flips exactly when the last CTA arrives (the low bits return to 0).
ES_DEV void soft_grid_sync(unsigned* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(ctr, inc);
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
            if (((old ^ cur) & 0x80000000u) == 0) __nanosleep(32);
        } while (((old ^ cur) & 0x80000000u) == 0);
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads, 1)
topn_cand_kernel(const double* __restrict__ s64, const int32_t* __restrict__ ids, int64_t n,
                 int id_mul, int id_add, int N, int cap, const uint32_t* __restrict__ hist_pre,
                 uint32_t* __restrict__ hist_g, int* __restrict__ out_count, double* __restrict__ out_s,
                 int32_t* __restrict__ out_id, long long* __restrict__ tr) {
    pdl_trigger();   // the union kernel may be scheduled now (it waits for this grid before reading);
                     // first, so that every CTA is resident before any later kernel (soft_grid_sync)
    pdl_wait();      // the scores / histogram of the scan (launched behind it with PDL)
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[2 * kNumSMs] = step_gtime();
    __shared__ uint32_t hist[kHistBins];
    __shared__ uint32_t warp_sum_s[kSelThreads / 32];
    __shared__ SelState st;
    __shared__ int found_bin, found_above, found_cnt, s_base;

    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    auto id_of = [&](int64_t i) -> int32_t { return ids ? ids[i] : (int32_t)(i * id_mul + id_add); };
    const int lane = lane_id(), wid = warp_id();

    if (threadIdx.x == 0) {
        for (int w = 0; w < 4; ++w) { st.pmask[w] = 0; st.pval[w] = 0; }
        st.remaining = N < 0 ? 0 : N;
        st.done = (N >= n) || (N <= 0);
    }
    __syncthreads();

    for (int pass = 0; pass < 12 && !st.done; ++pass) {
        int word, shift, nbits;
        pass_digit(pass, word, shift, nbits);
        const uint32_t dmask = (1u << nbits) - 1u;
        const uint32_t* hp;
        if (pass == 0 && hist_pre) {
            hp = hist_pre;
        } else {
            for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            SelState my = st;
            for (int64_t b0 = lo; b0 < hi; b0 += blockDim.x) {   // uniform trip count per warp
                const int64_t i = b0 + threadIdx.x;
                uint32_t digit = 0xFFFFFFFFu;
                if (i < hi && id_of(i) >= 0) {
                    SelWords k = sel_words(s64[i], id_of(i));
                    if (sel_matches(k, my)) digit = (k.w[word] >> shift) & dmask;
                }
                const unsigned peers = __match_any_sync(0xffffffffu, digit);
                if (digit != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[digit], (uint32_t)__popc(peers));
            }
            __syncthreads();
            uint32_t* hw = hist_g + (size_t)pass * kHistBins;
            for (int b = threadIdx.x; b < (1 << nbits); b += blockDim.x)
                if (hist[b]) atomicAdd(&hw[b], hist[b]);
            soft_grid_sync(hist_g + 12 * kHistBins);   // (the counter word after the 12 histograms)
            hp = hw;
        }
        // every CTA: the bin (descending) where the running count reaches `remaining`;
        // thread t owns bins [8t, 8t+8)
        constexpr int BPT = kHistBins / kSelThreads;
        uint32_t c[BPT], tot = 0;
        const int t = threadIdx.x;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const int b = BPT * t + j;
            c[j] = b < (1 << nbits) ? __ldcg(&hp[b]) : 0u;
            tot += c[j];
        }
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t v = __shfl_down_sync(0xffffffffu, inc, o);
            if (lane + o < 32) inc += v;
        }
        if (lane == 0) warp_sum_s[wid] = inc;
        __syncthreads();
        uint32_t above_w = 0;
        for (int w2 = wid + 1; w2 < kSelThreads / 32; ++w2) above_w += warp_sum_s[w2];
        const uint32_t rem = (uint32_t)st.remaining;
        uint32_t run = above_w + inc - tot;   // count in bins above this thread's range
#pragma unroll
        for (int j = BPT - 1; j >= 0; --j) {
            if (run < rem && run + c[j] >= rem) { found_bin = BPT * t + j; found_above = (int)run; found_cnt = (int)c[j]; }
            run += c[j];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int b = found_bin;
            const uint32_t in_bin = (uint32_t)found_cnt;
            const long long superset = (long long)(N - st.remaining) + found_above + in_bin;
            st.remaining -= found_above;
            st.pmask[word] |= dmask << shift;
            st.pval[word] |= ((uint32_t)b) << shift;
            // exact, or a candidate superset (everything in bins >= b) that fits
            if ((uint32_t)st.remaining == in_bin || superset <= cap) st.done = 1;
        }
        __syncthreads();
    }
    // compaction: appends of (s, id), one global atomic per CTA (a few hundred rows per
    // CTA: every row's load in flight, a block scan orders the CTA's appends); wider
    // slices take warp-aggregated appends
    SelState my = st;
    const bool take_all = (N >= n);
    constexpr int kCandIt = 4;
    if (hi - lo <= (int64_t)kCandIt * blockDim.x) {
        double sv[kCandIt];
        int32_t iv[kCandIt];
        bool sl[kCandIt];
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < kCandIt; ++u) {
            const int64_t i = lo + (int64_t)u * blockDim.x + threadIdx.x;
            sv[u] = 0.0;
            iv[u] = -1;
            if (i < hi) { sv[u] = s64[i]; iv[u] = id_of(i); }
        }
#pragma unroll
        for (int u = 0; u < kCandIt; ++u) {
            sl[u] = iv[u] >= 0 && (take_all || (N > 0 && sel_selected(sel_words(sv[u], iv[u]), my)));
            cnt += sl[u] ? 1 : 0;
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane == 31) warp_sum_s[wid] = (uint32_t)inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x / 32); ++w) { const int x = (int)warp_sum_s[w]; warp_sum_s[w] = tot; tot += x; }
            s_base = tot ? atomicAdd(out_count, tot) : 0;
        }
        __syncthreads();
        int o = s_base + (int)warp_sum_s[wid] + inc - cnt;
#pragma unroll
        for (int u = 0; u < kCandIt; ++u)
            if (sl[u]) {
                if (o < cap) { out_s[o] = sv[u]; out_id[o] = iv[u]; }
                ++o;
            }
        if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[2 * kNumSMs + 1] = step_gtime();
        return;
    }
    for (int64_t b0 = lo; b0 < hi; b0 += blockDim.x) {
        const int64_t i = b0 + threadIdx.x;
        bool sel = false;
        double s = 0.0;
        int32_t id = 0;
        if (i < hi) {
            s = s64[i];
            id = id_of(i);
            sel = id >= 0 && (take_all || (N > 0 && sel_selected(sel_words(s, id), my)));
        }
        const unsigned m = __ballot_sync(0xffffffffu, sel);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(out_count, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int o = base + __popc(m & ((1u << lane) - 1u));
        if (sel && o < cap) { out_s[o] = s; out_id[o] = id; }
    }
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[2 * kNumSMs + 1] = step_gtime();
}

cudaError_t launch_topn_cand(const double* s64, const int32_t* ids, int64_t n, int id_mul, int id_add,
                             int N, int cap, const uint32_t* hist_pre, uint32_t* hist_g, int* out_count,
                             double* out_s, int32_t* out_id, cudaStream_t st, bool prezeroed) {
    if (!prezeroed) {   // (the scan zeroes them when it directly precedes this selection)
        cudaMemsetAsync(hist_g, 0, 12 * kHistBins * sizeof(uint32_t), st);
        cudaMemsetAsync(out_count, 0, sizeof(int), st);
    }
    int grid = kNumSMs;
    if (n < (int64_t)grid * 64) grid = (int)((n + 63) / 64);
    if (grid < 1) grid = 1;
    // programmatic: its CTAs take the SMs the scan's CTAs leave and wait there, and the
    // union behind it may be scheduled early (the rare multi-pass path syncs the grid
    // with soft_grid_sync: hist_g holds 12 * kHistBins + 1 words)
    return launch_pdl(topn_cand_kernel, dim3(grid), dim3(kSelThreads), 0, st, s64, ids, n, id_mul, id_add, N,
                           cap, hist_pre, hist_g, out_count, out_s, out_id, s_step_trace);
}

}  // namespace es
