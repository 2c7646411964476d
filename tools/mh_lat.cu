// mh_lat.cu — per-phase cycle profile of the MH window kernel (window.cu built with
// MH_PROFILE): block 0 / thread 0 accumulates clock64 deltas between the step's phases.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//        -I paper_1506_05741_b200/csrc tools/mh_lat.cu -o tools/mh_lat && tools/mh_lat [d] [chains]
#define MH_PROFILE 1
#include <map>
#include <vector>
#include <cstdio>
#include <mutex>
#include "window.cu"

namespace dgb {
std::atomic<uint64_t> g_launch_count{0};
thread_local uint64_t t_launch_count = 0;
bool sync_check_enabled() { return false; }
void set_smem_attr(const void* f, int bytes) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
}  // namespace dgb

using namespace dgb;

int main(int argc, char** argv) {
    const int d = argc > 1 ? atoi(argv[1]) : 1024, C = argc > 2 ? atoi(argv[2]) : 64, L = d / 2;
    const int64_t ld = (d + 7) / 8 * 8, win = (int64_t)L * ld;
    std::vector<double> h((size_t)C * win);
    srand(3);
    auto rnd = [] { return (rand() / (double)RAND_MAX - 0.5) * 0.02; };
    double *W, *Xi, *H, *g, *y, *lp, *qd, *beta, *ie, *bc;
    uint64_t *nacc, *uctr;
    int *kcount, *acnt, *src, *mult;
    PhiloxKey* keys;
    cudaMalloc(&W, h.size() * 8);
    cudaMalloc(&Xi, h.size() * 8);
    cudaMalloc(&H, h.size() * 8);
    for (auto& v : h) v = rnd();
    cudaMemcpy(W, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(Xi, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(H, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&g, C * ld * 8);
    cudaMalloc(&y, C * ld * 8);
    cudaMalloc(&ie, ld * 8);
    cudaMalloc(&bc, ld * 8);
    std::vector<double> ones(ld, 1.0);
    cudaMemcpy(ie, ones.data(), ld * 8, cudaMemcpyHostToDevice);
    cudaMemset(bc, 0, ld * 8);
    cudaMemset(g, 0, C * ld * 8);
    cudaMemset(y, 0, C * ld * 8);
    cudaMalloc(&lp, C * 8);
    cudaMalloc(&qd, C * 8);
    cudaMalloc(&beta, C * 8);
    cudaMemset(lp, 0, C * 8);
    cudaMemset(qd, 0, C * 8);
    std::vector<double> b(C, 0.3);
    cudaMemcpy(beta, b.data(), C * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&nacc, C * 8);
    cudaMalloc(&uctr, C * 8);
    cudaMemset(nacc, 0, C * 8);
    cudaMemset(uctr, 0, C * 8);
    cudaMalloc(&kcount, C * 4);
    cudaMalloc(&acnt, C * 4);
    cudaMalloc(&src, (size_t)C * L * 4);
    cudaMalloc(&mult, (size_t)C * L * 4);
    std::vector<PhiloxKey> k(C);
    for (int i = 0; i < C; ++i) k[i] = make_philox_key(7, i, "uniform");
    cudaMalloc(&keys, C * sizeof(PhiloxKey));
    cudaMemcpy(keys, k.data(), C * sizeof(PhiloxKey), cudaMemcpyHostToDevice);
    StepParams p{};
    p.d = d;
    p.n_lag = L;
    p.chains = C;
    p.ld = ld;
    p.win_stride = win;
    p.dg = d;
    p.ldg = ld;
    p.hwin_stride = win;
    p.W = W;
    p.Xi = Xi;
    p.H = H;
    p.first = 0;
    p.kcount = kcount;
    p.acc_count = acnt;
    p.state_src = src;
    p.state_mult = mult;
    p.g = g;
    p.y = y;
    p.log_pi = lp;
    p.quad = qd;
    p.beta = beta;
    p.n_accepted = nacc;
    p.ukeys = keys;
    p.uctr = uctr;
    p.infl = 1.0;
    p.pcn = 1;
    p.inv_eig = ie;
    p.bcoef = bc;
    p.out_ld = L;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch_mh_window(p, 0);
    cudaDeviceSynchronize();
    std::vector<long long> z(8, 0);
    cudaMemcpyToSymbol(g_mh_prof, z.data(), 64);
    cudaEventRecord(e0);
    launch_mh_window(p, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> pr(8);
    cudaMemcpyFromSymbol(pr.data(), g_mh_prof, 64);
    const char* names[] = {"loop top (logu, stage index)", "mbar_wait", "candidate + dots", "warp_sum2 + STS",
                           "BAR.SYNC", "refill issue + cross-warp sum", "decision, adoption, stores"};
    long long tot = 0;
    for (int i = 0; i < 7; ++i) tot += pr[i];
    printf("d=%d chains=%d n_lag=%d: %.3f ms, %.0f cycles/step (block 0)\n", d, C, L, ms, (double)tot / L);
    for (int i = 0; i < 7; ++i) printf("  %-32s %7.1f cycles/step\n", names[i], (double)pr[i] / L);
    printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
