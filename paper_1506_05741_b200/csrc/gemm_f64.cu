// gemm_f64.cu — batched FP64 DMMA GEMM (see gemm_f64.cuh for the contract; the tile
// itself is gemm_tile.cuh, shared with the persistent Cholesky kernel).
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
    const int M = p.m_vec ? min(p.M, p.m_vec[b]) : p.M;
    if (n0 >= p.N || m0 >= M) return;
    if (p.tri_c_lower && n0 > m0 + CF::BM - 1) return;
    extern __shared__ __align__(16) double smem[];
    int K = p.k_vec ? p.k_vec[b] : p.K;
    if (p.tri_b_lower) K = min(K, n0 + CF::BN);
    double alpha = p.alpha;
    if (p.alpha_vec) alpha *= p.alpha_vec[b] * p.alpha_vec_mul;
    tile::gemm_tile<CF, AK, BKM>(p.A[b] + p.a_off, p.B[b] + p.b_off, p.C[b] + p.c_off, p.lda, p.ldb, p.ldc, M, p.N, K,
                                 m0, n0, alpha, p.beta, p.tri_c_lower != 0, smem, p.tri_b_lower != 0);
}

template <class CF, bool AK, bool BKM>
void launch(const GemmBatch& g, int batch, cudaStream_t stream) {
    auto kern = gemm_f64_kernel<CF, AK, BKM>;
    set_smem_attr(reinterpret_cast<const void*>(kern), CF::SMEM_BYTES);
    dim3 grid((unsigned)ceil_div(g.N, CF::BN), (unsigned)ceil_div(g.M, CF::BM), (unsigned)batch);
    kern<<<grid, CF::THREADS, CF::SMEM_BYTES, stream>>>(g);
    DGB_LAUNCH_CHECK();
    count_launch();
}

// One tile configuration for every product (tools/gemm_k_sweep.py: C = A B, 32768 x 1024,
// K = 512 / 1024, % of the live DMMA peak): 128x64 tiles, 8 warps of 32x32, 32-deep K
// stages double-buffered, 2 CTAs per SM -- beta=0 86.9 / 89.4%, beta=1 85.5 / 88.4%.
// Measured and dropped (round 1): 128x128 tiles with 1 CTA/SM (9% slower per batch), 4
// warps of 64x32 in a 3-deep ring of 16-deep stages (equal in the engine), 16-deep stages
// (1.2% slower), 64x128 tiles of 4 warps of 32x64.
template <bool AK, bool BKM>
using GemmCfgT = Cfg<128, 64, 32, 2, AK, BKM, 4, 2, 2>;

}  // namespace

// 64 x 64 tiles, 4 warps of 32 x 32, up to 3 CTAs per SM: half the long-K latency of one tile
// (the factorization's left-looking updates sit on the refactor's critical path)
template <bool AK, bool BKM>
using GemmCfgS = Cfg<64, 64, 32, 2, AK, BKM, 2, 2, 3>;

void gemm_f64_small(const GemmBatch& g, int batch, cudaStream_t stream) {
    if (batch <= 0 || g.M <= 0 || g.N <= 0) return;
    launch<GemmCfgS<true, true>, true, true>(g, batch, stream);
}

void gemm_f64(const GemmBatch& g, int batch, bool a_kmajor, bool b_kmajor, cudaStream_t stream) {
    if (batch <= 0 || g.M <= 0 || g.N <= 0) return;
    if (a_kmajor && b_kmajor) launch<GemmCfgT<true, true>, true, true>(g, batch, stream);
    else if (a_kmajor && !b_kmajor) launch<GemmCfgT<true, false>, true, false>(g, batch, stream);
    else if (!a_kmajor && b_kmajor) launch<GemmCfgT<false, true>, false, true>(g, batch, stream);
    else launch<GemmCfgT<false, false>, false, false>(g, batch, stream);
}

}  // namespace dgb
