// TMA staging lab: checks the tensor-map view of the packed 128 x 128 tile slots and the
// swizzled shared-memory fragment addressing that update_phase uses (kernels.cu), in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_lab tools/tma_lab.cu && /tmp/tma_lab
// One 3-D tensor map per operand role over a slot array (column-major slots, ld 128):
//   dim0 = 8 consecutive rows (8 B stride), dim1 = column over all slots (1 KB stride),
//   dim2 = row group of 8 (64 B stride).
// L chunk (128 rows x 32 k): box {8, 32, 16} at (0, slot*128 + k0, 0)   -> off = G*2048 + k*64 + r8*8
// R chunk (32 k x 128 cols): box {8, 128, 4} at (0, slot*128, k0/8)     -> off = KG*8192 + n*64 + k8*8
// both with SWIZZLE_64B (byte-address bits 4-5 ^= bits 7-8).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return nullptr;
    return (EncodeFn)fn;
}

static bool make_map(EncodeFn enc, CUtensorMap* m, double* base, size_t nslots, int b1, int b2) {
    const cuuint64_t dims[3] = {8, (cuuint64_t)nslots * 128, 16};
    const cuuint64_t strides[2] = {1024, 64};
    const cuuint32_t box[3] = {8, (cuuint32_t)b1, (cuuint32_t)b2};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed: %d\n", (int)r);
    return r == CUDA_SUCCESS;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(512, 1) k_lab(const __grid_constant__ CUtensorMap mapL,
                                                 const __grid_constant__ CUtensorMap mapR,
                                                 const double* slots, int slotL, int slotR, int k0,
                                                 int* bad) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    unsigned char* sL = smem;
    unsigned char* sR = smem + 32768;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3, wm = warp >> 2, wn = warp & 3;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(65536) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(smem_u32(sL)), "l"(&mapL), "r"(0), "r"(slotL * 128 + k0), "r"(0), "r"(smem_u32(&bar)) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(smem_u32(sR)), "l"(&mapR), "r"(0), "r"(slotR * 128), "r"(k0 / 8), "r"(smem_u32(&bar)) : "memory");
    }
    {
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    }
    // fragment addressing of mma_chunk: two base offsets per operand (kk % 8 == 0 / == 4)
    const int s = (g >> 1) & 3;
    const unsigned a0 = wm * 8192 + q * 64 + ((g * 8) ^ ((q >> 1) << 4));
    const unsigned a1 = wm * 8192 + q * 64 + ((g * 8) ^ (((q >> 1) | 2) << 4));
    const unsigned b0 = (wn * 32 + g) * 64 + ((q * 8) ^ (s << 4));
    const unsigned b1 = (wn * 32 + g) * 64 + (((4 + q) * 8) ^ (s << 4));
    int nbad = 0;
    const double* L = slots + (size_t)slotL * 16384;
    const double* R = slots + (size_t)slotR * 16384;
    for (int kk = 0; kk < 32; kk += 4) {
        for (int mi = 0; mi < 4; ++mi) {
            const double v = *(const double*)(sL + ((kk & 4) ? a1 : a0) + mi * 2048 + kk * 64);
            const double e = L[(wm * 32 + mi * 8 + g) + (size_t)(k0 + kk + q) * 128];
            if (v != e) ++nbad;
        }
        for (int ni = 0; ni < 4; ++ni) {
            const double v = *(const double*)(sR + ((kk & 4) ? b1 : b0) + ni * 512 + (kk >> 3) * 8192);
            const double e = R[(k0 + kk + q) + (size_t)(wn * 32 + ni * 8 + g) * 128];
            if (v != e) ++nbad;
        }
    }
    // the addressing update_phase uses: the four k of a DMMA step are {0, 1, 4, 5} (step 0) and
    // {2, 3, 6, 7} (step 1) of each group of eight, which makes the loads conflict-free
    const int kq = (q & 1) + 4 * (q >> 1);
    const unsigned pa[2] = {wm * 8192u + kq * 64 + ((g * 8) ^ ((2 * (q >> 1)) << 4)),
                            wm * 8192u + (kq + 2) * 64 + ((g * 8) ^ ((1 + 2 * (q >> 1)) << 4))};
    const unsigned pb[2] = {(wn * 32u + g) * 64 + ((kq * 8) ^ (s << 4)),
                            (wn * 32u + g) * 64 + (((kq + 2) * 8) ^ (s << 4))};
    for (int kk = 0; kk < 32; kk += 4) {
        const int step = (kk >> 2) & 1, k = (kk >> 3) * 8 + 2 * step + kq;
        for (int mi = 0; mi < 4; ++mi) {
            const double v = *(const double*)(sL + pa[step] + mi * 2048 + (kk >> 3) * 512);
            if (v != L[(wm * 32 + mi * 8 + g) + (size_t)(k0 + k) * 128]) ++nbad;
        }
        for (int ni = 0; ni < 4; ++ni) {
            const double v = *(const double*)(sR + pb[step] + ni * 512 + (kk >> 3) * 8192);
            if (v != R[(k0 + k) + (size_t)(wn * 32 + ni * 8 + g) * 128]) ++nbad;
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

int main() {
    EncodeFn enc = get_encode();
    if (!enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    const size_t nslots = 5;
    std::vector<double> h(nslots * 16384);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i + 0.25;
    double* d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    int* bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    CUtensorMap mL, mR;
    if (!make_map(enc, &mL, d, nslots, 32, 16) || !make_map(enc, &mR, d, nslots, 128, 4)) return 2;
    cudaFuncSetAttribute(k_lab, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    int total = 0;
    for (int k0 = 0; k0 < 128; k0 += 32) {
        k_lab<<<1, 512, 65536 + 1024>>>(mL, mR, d, 1 + (k0 / 32) % 3, 4 - (k0 / 32) % 3, k0, bad);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("kernel error: %s\n", cudaGetErrorString(e));
            return 3;
        }
    }
    cudaMemcpy(&total, bad, 4, cudaMemcpyDeviceToHost);
    printf("tma_lab: mismatches = %d %s\n", total, total == 0 ? "OK" : "FAIL");
    return total != 0;
}
