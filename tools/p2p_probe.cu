// p2p_probe.cu -- NVLink peer-write bandwidth probe for the fused global-qubit swap.
// Two GPUs in one process (peer access enabled); both directions run at once, as in the swap.
// Variants (each moves `bytes` from a local buffer into the peer's buffer):
//   st16     : 16-byte st.global per thread, fully contiguous
//   st16row  : 16-byte stores in 128-byte rows scattered with a 2 MiB stride (run-set pattern)
//   bulk     : cp.async.bulk global->smem, then cp.async.bulk smem->peer global (TMA engine)
//   ce       : cudaMemcpyPeerAsync (copy engines)
//   local    : st16 into the local second buffer (HBM copy reference)
//   splitS   : 16-byte stores, chunks of S bytes alternate between the peer and the local second
//              buffer (the low-bit global-qubit swap: S = 64 / 32 / 16 B at G = 2 / 4 / 8);
//              GBps_per_dir counts the peer half only
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe tools/p2p_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__global__ void st16(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(dst + i, __ldcs(src + i));
}

// rows of 8 amplitudes (128 B); row r of a "tile" of 512 rows goes to (tile, r) with row stride 2 MiB
__global__ void st16row(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t n) {
    const size_t rows = n / 8;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t row = i >> 3, e = i & 7;
        // permute rows: row = t*512 + r  ->  r*(rows/512) + t
        const size_t t = row >> 9, r = row & 511;
        const size_t drow = r * (rows >> 9) + t;
        __stcs(dst + drow * 8 + e, __ldcs(src + i));
    }
}

template <int LOGC>  // chunk = 2^LOGC amplitudes
__global__ void split(const double2 *__restrict__ src, double2 *__restrict__ peer, double2 *__restrict__ loc,
                      size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double2 v = __ldcs(src + i);
        if ((i >> LOGC) & 1) __stcs(peer + i, v);
        else __stcs(loc + i, v);
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// one CTA moves chunks of CH bytes: bulk load into smem (mbarrier), bulk store to dst
template <int CH>
__global__ void bulk(const char *__restrict__ src, char *__restrict__ dst, size_t bytes) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const size_t nch = bytes / CH;
    int s = 0;
    uint32_t ph[2] = {0, 0};
    size_t c = blockIdx.x;
    // prologue: issue first load
    auto issue = [&](size_t cc, int st) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(CH));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + st * CH)),
            "l"(src + cc * CH), "r"(CH), "r"(smem_u32(&bar[st]))
            : "memory");
    };
    if (c < nch) issue(c, 0);
    for (; c < nch; c += gridDim.x) {
        const size_t nx = c + gridDim.x;
        if (nx < nch) {
            // stage s^1 must be free: its previous store has finished reading smem
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            issue(nx, s ^ 1);
        }
        // wait load of stage s
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&bar[s])), "r"(ph[s]));
        }
        ph[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH),
                     "r"(smem_u32(sm + s * CH)), "r"(CH)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        s ^= 1;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
    size_t bytes = (argc > 1 ? strtoull(argv[1], 0, 10) : 4096ull) << 20;
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    if (ng < 2) {
        printf("{\"error\": \"need 2 GPUs\"}\n");
        return 0;
    }
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, 0, 1));
    printf("# peer access 0->1: %d\n", can);
    double2 *src[2], *dst[2], *loc[2];
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(d ^ 1, 0));
        CK(cudaMalloc(&src[d], bytes));
        CK(cudaMalloc(&dst[d], bytes));
        CK(cudaMalloc(&loc[d], bytes));
        CK(cudaMemset(src[d], 1, bytes));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
        CK(cudaFuncSetAttribute(bulk<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768));
        CK(cudaFuncSetAttribute(bulk<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536));
    }
    const size_t n = bytes / 16;
    const char *names[] = {"st16", "st16row", "bulk32k", "bulk64k", "bulk32k_x2", "ce", "local_st16", "st16_1dir",
                           "bulk64k_1dir", "ce_1dir", "split64", "split32", "split16", "split128"};
    for (int v = 0; v < 14; ++v) {
        if (argc > 2 && v < 10) continue;  // second argument: split variants only
        for (int grid_mul = 1; grid_mul <= ((v == 0 || v == 1 || v == 6) ? 4 : 1); grid_mul *= 2) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                for (int d = 0; d < 2; ++d) {
                    CK(cudaSetDevice(d));
                    CK(cudaDeviceSynchronize());
                }
                for (int d = 0; d < 2; ++d) {
                    const bool onedir = (v >= 7);
                    if (onedir && d == 1) continue;
                    CK(cudaSetDevice(d));
                    CK(cudaEventRecord(e0[d], st[d]));
                    double2 *to = (v == 6) ? loc[d] : dst[d ^ 1];
                    switch (v) {
                        case 0:
                        case 6:
                        case 7: st16<<<sms * 2 * grid_mul, 512, 0, st[d]>>>(src[d], to, n); break;
                        case 1: st16row<<<sms * 2 * grid_mul, 512, 0, st[d]>>>(src[d], to, n); break;
                        case 2: bulk<32768><<<sms, 32, 2 * 32768, st[d]>>>((const char *)src[d], (char *)to, bytes); break;
                        case 3:
                        case 8: bulk<65536><<<sms, 32, 2 * 65536, st[d]>>>((const char *)src[d], (char *)to, bytes); break;
                        case 4: bulk<32768><<<sms * 2, 32, 2 * 32768, st[d]>>>((const char *)src[d], (char *)to, bytes); break;
                        case 5:
                        case 9: CK(cudaMemcpyPeerAsync(to, d ^ 1, src[d], d, bytes, st[d])); break;
                        case 10: split<2><<<sms * 2, 512, 0, st[d]>>>(src[d], to, loc[d], n); break;
                        case 11: split<1><<<sms * 2, 512, 0, st[d]>>>(src[d], to, loc[d], n); break;
                        case 12: split<0><<<sms * 2, 512, 0, st[d]>>>(src[d], to, loc[d], n); break;
                        case 13: split<3><<<sms * 2, 512, 0, st[d]>>>(src[d], to, loc[d], n); break;
                    }
                    CK(cudaGetLastError());
                    CK(cudaEventRecord(e1[d], st[d]));
                }
                float ms = 0;
                for (int d = 0; d < 2; ++d) {
                    if (v >= 7 && d == 1) continue;
                    CK(cudaSetDevice(d));
                    CK(cudaEventSynchronize(e1[d]));
                    float t = 0;
                    CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
                    if (t > ms) ms = t;
                }
                if (rep > 0 && ms < best) best = ms;
            }
            printf("{\"variant\": \"%s\", \"grid_mul\": %d, \"bytes\": %zu, \"ms\": %.3f, \"GBps_per_dir\": %.1f}\n",
                   names[v], grid_mul, bytes, best, (v >= 10 ? 0.5 : 1.0) * bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
