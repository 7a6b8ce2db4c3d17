// gather_probe.cu -- measured ceiling for random sector gathers on one B200.
//
// The walk path is a stream of independent random 16-32 B reads (node record,
// rejection-trial edge record, hash bucket).  The copy bandwidth in
// MEASURED_PEAKS.json is a sequential ceiling; this probe measures what HBM3e
// delivers when every request is a random location of a buffer far larger
// than L2, per request size and per load flavour (cache operator / L2 policy),
// so the DRAM bytes each flavour moves per request can be read off ncu.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather_probe tools/gather_probe.cu
//   tools/bin/gather_probe [buffer GiB] [L2 fetch granularity] > profiles/<round>_gather_probe.json
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

// Load flavours for one 16 B random read.
enum Flavor { F_NC = 0, F_CG, F_CS, F_CV, F_LU, F_EVICT_FIRST, F_NOALLOC, F_CPASYNC, F_PF64, F_NUM };
static const char* kFlavorName[F_NUM] = {
    "ld.global.nc", "ld.global.cg", "ld.global.cs", "ld.global.cv", "ld.global.lu",
    "ld.global.nc.L2::cache_hint(evict_first)", "ld.global.nc.L1::no_allocate",
    "cp.async.cg.shared.global 16", "ld.global.nc.L2::64B"};

template <int F>
__device__ __forceinline__ uint32_t load16(const uint4* p, uint64_t pol, uint4* smem) {
    uint32_t a, b, c, d;
    if (F == F_NC) {
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else if (F == F_CG) {
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else if (F == F_CS) {
        asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else if (F == F_CV) {
        asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else if (F == F_LU) {
        asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else if (F == F_EVICT_FIRST) {
        asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p), "l"(pol));
    } else if (F == F_NOALLOC) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else if (F == F_PF64) {
        asm volatile("ld.global.nc.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    } else {  // F_CPASYNC: caller waits and reads smem
        const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(p) : "memory");
        return 0;
    }
    return a ^ d;
}

// K independent random 16 B requests per thread per iteration; the next
// batch's addresses depend on this batch's data (a chain, like a walk).
template <int F, int K>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ buf, uint32_t lg16,
                                             int iters, uint32_t* sink) {
    __shared__ uint4 s_land[K][256];
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t pol = 0;
    if (F == F_EVICT_FIRST) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint64_t st = tid * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            const uint64_t slot = (st ^ (st >> 29)) >> (64 - lg16);  // power-of-two buffer
            v[k] = load16<F>(buf + slot, pol, &s_land[k][threadIdx.x]);
        }
        if (F == F_CPASYNC) {
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = s_land[k][threadIdx.x].x ^ s_land[k][threadIdx.x].w;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) acc += v[k];
        st ^= acc & 1;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int F, int K>
void run(const uint4* buf, uint32_t lg16, uint32_t* sink, int sms, bool first) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int iters = 64;
    const int blocks = sms * 4;
    gather<F, K><<<blocks, 256>>>(buf, lg16, iters, sink);  // warm
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) gather<F, K><<<blocks, 256>>>(buf, lg16, iters, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double req = 5.0 * blocks * 256.0 * iters * K;
    const double rps = req / (ms * 1e-3);
    printf("%s  {\"flavor\": \"%s\", \"bytes\": 16, \"inflight_per_thread\": %d, \"grid\": %d, "
           "\"requests_per_s\": %.4g, \"useful_gbs\": %.1f}",
           first ? "" : ",\n", kFlavorName[F], K, blocks, rps, rps * 16 / 1e9);
    CK(cudaEventDestroy(a));
    CK(cudaEventDestroy(b));
}

int main(int argc, char** argv) {
    const int lgbytes = argc > 1 ? atoi(argv[1]) : 32;  // log2 buffer bytes (32 = 4 GiB)
    const uint32_t lg16 = lgbytes - 4;
    const uint64_t bytes = 1ull << lgbytes;
    uint4* buf;
    uint32_t* sink;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 1, bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    if (argc > 2) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(argv[2])));
    size_t gran = 0;
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    printf("{\"probe\": \"random 16 B gathers over a %llu MiB buffer (L2 126 MB)\", \"sms\": %d, "
           "\"l2_fetch_granularity\": %zu, \"results\": [\n",
           (unsigned long long)(bytes >> 20), sms, gran);
    run<F_NC, 4>(buf, lg16, sink, sms, true);
    run<F_CG, 4>(buf, lg16, sink, sms, false);
    run<F_CS, 4>(buf, lg16, sink, sms, false);
    run<F_CV, 4>(buf, lg16, sink, sms, false);
    run<F_LU, 4>(buf, lg16, sink, sms, false);
    run<F_EVICT_FIRST, 4>(buf, lg16, sink, sms, false);
    run<F_NOALLOC, 4>(buf, lg16, sink, sms, false);
    run<F_CPASYNC, 4>(buf, lg16, sink, sms, false);
    run<F_PF64, 4>(buf, lg16, sink, sms, false);
    run<F_NC, 1>(buf, lg16, sink, sms, false);
    run<F_NC, 8>(buf, lg16, sink, sms, false);
    printf("\n]}\n");
    return 0;
}
