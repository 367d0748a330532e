// common.cuh -- small device helpers shared by the libevospec kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <utility>

#define ES_DEV __device__ __forceinline__

namespace es {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

ES_DEV float bf16_bits_to_f32(uint32_t b16) { return __uint_as_float(b16 << 16); }

// 16-byte streaming load that does not allocate in L1 (read-once data).
ES_DEV uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// Unpack 8 bf16 (one uint4) into fp32.
ES_DEV void unpack_bf16x8(const uint4& u, float (&f)[8]) {
    f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
    f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
    f[4] = __uint_as_float(u.z << 16); f[5] = __uint_as_float(u.z & 0xFFFF0000u);
    f[6] = __uint_as_float(u.w << 16); f[7] = __uint_as_float(u.w & 0xFFFF0000u);
}

// Monotone map float -> uint32: a > b  <=>  key(a) > key(b) (no NaN inputs).
ES_DEV uint32_t float_key(float f) {
    if (f == 0.0f) f = 0.0f;  // canonical +0
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// Monotone map double -> uint64.
ES_DEV uint64_t double_key(double x) {
    if (x == 0.0) x = 0.0;
    uint64_t u = (uint64_t)__double_as_longlong(x);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// (a, ida) precedes (b, idb) under the order (value desc, id asc).
template <typename T>
ES_DEV bool before(T a, int ida, T b, int idb) { return a > b || (a == b && ida < idb); }

ES_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
ES_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
ES_DEV double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
ES_DEV int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp arg-best under (value desc, key asc); every lane gets the winner.
ES_DEV void warp_argbest(float& v, int& key) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, v, o);
        int ok = __shfl_xor_sync(0xffffffffu, key, o);
        if (before(ov, ok, v, key)) { v = ov; key = ok; }
    }
}

ES_DEV int lane_id() { return threadIdx.x & 31; }

// Programmatic dependent launch: a kernel launched with launch_pdl() may start
// while its predecessor drains; it must pdl_wait() before touching the
// predecessor's outputs. pdl_trigger() lets the successor be scheduled early.
ES_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
ES_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// launch_pdl for a cooperative grid (grid-wide sync): programmatic serialization
// and co-residency together
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                   Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
ES_DEV int warp_id() { return threadIdx.x >> 5; }
ES_DEV long long globaltimer_ns() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
ES_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

}  // namespace es
