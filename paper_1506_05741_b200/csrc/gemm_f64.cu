// gemm_f64.cu — batched FP64 DMMA GEMM (see gemm_f64.cuh for the contract; the tile
// itself is gemm_tile.cuh, shared with the persistent Cholesky kernel).
#include <cstdlib>

#include "gemm_f64.cuh"
#include "gemm_tile.cuh"

namespace dgb {

namespace {

using tile::Cfg;

template <class CF, bool AK, bool BKM>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB) gemm_f64_kernel(GemmBatch p) {
    const int b = blockIdx.z;
    if (p.active && !p.active[b]) return;
    // triangular B: tile n has K = (n+1) BN, so hand out the longest tiles first
    // (longest-processing-time order shortens the tail of the launch)
    const int nt = p.tri_b_lower ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
    const int n0 = nt * CF::BN;
    const int m0 = blockIdx.y * CF::BM;
    if (n0 >= p.N || m0 >= p.M) return;
    if (p.tri_c_lower && n0 > m0 + CF::BM - 1) return;
    extern __shared__ __align__(16) double smem[];
    int K = p.K;
    if (p.tri_b_lower) K = min(K, n0 + CF::BN);
    double alpha = p.alpha;
    if (p.alpha_vec) alpha *= p.alpha_vec[b] * p.alpha_vec_mul;
    tile::gemm_tile<CF, AK, BKM>(p.A[b] + p.a_off, p.B[b] + p.b_off, p.C[b] + p.c_off, p.lda, p.ldb, p.ldc, p.M, p.N,
                                 K, m0, n0, alpha, p.beta, p.tri_c_lower != 0, smem, p.tri_b_lower != 0);
}

template <class CF, bool AK, bool BKM>
void launch(const GemmBatch& g, int batch, cudaStream_t stream) {
    auto kern = gemm_f64_kernel<CF, AK, BKM>;
    static bool attr_set = false;  // per template instance
    if (!attr_set) {
        DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES));
        attr_set = true;
    }
    dim3 grid((unsigned)ceil_div(g.N, CF::BN), (unsigned)ceil_div(g.M, CF::BM), (unsigned)batch);
    kern<<<grid, CF::THREADS, CF::SMEM_BYTES, stream>>>(g);
    DGB_LAUNCH_CHECK();
    count_launch();
}

template <bool AK, bool BKM>
void dispatch_shape(const GemmBatch& g, int batch, cudaStream_t stream, GemmShape shape) {
    // Tile configurations (tools/gemm_k_sweep.py: C = A B, 32768 x 1024, K = 512 / 1024,
    // % of the live DMMA peak; the next stage's copies issued behind the first DMMAs):
    //   2  128x64 tiles, 8 warps of 32x32, 32-deep K stages double-buffered, 2 CTAs/SM:
    //      beta=0 86.9 / 89.4%, beta=1 85.5 / 88.4%; the default for every shape
    //   4  128x64 tiles, 4 warps of 64x32 (half the fragment loads per DMMA), 16-deep
    //      stages in a 3-deep ring, 2 CTAs/SM: beta=0 86.3 / 88.9%, beta=1 83.7 / 87.6%
    //      (better than 2 before the copy-issue move; equal in the engine since)
    //   1  as 2 with 16-deep stages in a 3-deep ring (1.2% slower per batch)
    //   0  128x128 (Big) / 128x64 (Narrow) tiles, 1 CTA/SM, 16-deep 4-deep ring (9% slower)
    // Measured and dropped: 64x128 tiles of 4 warps of 32x64 (16- or 32-deep), 4 warps
    // with 32-deep double-buffered stages, 128x128 with 32-deep stages (1 CTA/SM).
    // For reference, cuBLAS's FP64 GEMM on this GPU is an sm80 CUTLASS kernel (64x128
    // tiles, 4 warps, 16-deep 3-stage ring, 2 CTAs/SM): 96.5% tensor-pipe active at 8192^3.
    // DIAM_B200_GEMM_CFG forces one configuration for every shape but Square.
    static const int cfg = [] {
        const char* e = std::getenv("DIAM_B200_GEMM_CFG");
        return e ? std::atoi(e) : -1;
    }();
    const int c = cfg >= 0 ? cfg : 2;
    if (shape == GemmShape::Square) {
        launch<Cfg<128, 128, 16, 4, AK, BKM>, AK, BKM>(g, batch, stream);
        return;
    }
    if (c == 2) {
        launch<Cfg<128, 64, 32, 2, AK, BKM, 4, 2, 2>, AK, BKM>(g, batch, stream);
        return;
    }
    if (c == 4) {
        launch<Cfg<128, 64, 16, 3, AK, BKM, 2, 2, 2>, AK, BKM>(g, batch, stream);
        return;
    }
    if (c == 1) {
        launch<Cfg<128, 64, 16, 3, AK, BKM, 4, 2, 2>, AK, BKM>(g, batch, stream);
        return;
    }
    if (shape == GemmShape::Narrow)
        launch<Cfg<128, 64, 16, 4, AK, BKM>, AK, BKM>(g, batch, stream);
    else
        launch<Cfg<128, 128, 16, 4, AK, BKM>, AK, BKM>(g, batch, stream);
}

}  // namespace

void gemm_f64(const GemmBatch& g, int batch, bool a_kmajor, bool b_kmajor, cudaStream_t stream,
              GemmShape shape) {
    if (batch <= 0 || g.M <= 0 || g.N <= 0) return;
    if (a_kmajor && b_kmajor) dispatch_shape<true, true>(g, batch, stream, shape);
    else if (a_kmajor && !b_kmajor) dispatch_shape<true, false>(g, batch, stream, shape);
    else if (!a_kmajor && b_kmajor) dispatch_shape<false, true>(g, batch, stream, shape);
    else dispatch_shape<false, false>(g, batch, stream, shape);
}

}  // namespace dgb
