// checkpoint.cu — DIAMCKPT v1 save/restore of the GPU engine state.
//
// Layout: proj/src/runner.cpp:398-457 (writer) and :139-207 (reader), field by field,
// so a checkpoint written here is readable by the reference and vice versa; the
// engine state lives on the device and is staged through host memory. After the
// reference's fields we append a "B200EXT1" block with each chain's
// y = L^-1 (x - x_ref): the step recursion carries y exactly, so restoring it
// (instead of re-solving) makes a resumed run continue bit-for-bit.
#include <cmath>
#include <cstring>

#include "engine.hpp"

namespace dgb {

namespace {

constexpr char kCkptMagic[8] = {'D', 'I', 'A', 'M', 'C', 'K', 'P', 'T'};
constexpr char kExtMagic[8] = {'B', '2', '0', '0', 'E', 'X', 'T', '1'};
// the engine's whitened state exactly (the reference's x-space fields are its image through
// G^-1, which a resume could only invert to rounding): global S_z / m_z, then per chain L_z,
// [L_z^-1], S_z, [cumulative S_z], m_z, the x-space raw diagonal, the cumulative one
constexpr char kExt2Magic[8] = {'B', '2', '0', '0', 'E', 'X', 'T', '2'};
constexpr uint32_t kVersion = 1;
constexpr uint32_t kEndian = 0x01020304u;

void write_opt(BinOut& w, const std::optional<double>& v) {
    w.pod<uint32_t>(v ? 1 : 0);
    w.pod<double>(v.value_or(0.0));
}

std::optional<double> read_opt(BinIn& r) {
    const bool has = r.pod<uint32_t>() != 0;
    const double v = r.pod<double>();
    return has ? std::optional<double>(v) : std::nullopt;
}

// KernelConfig (proj/src/runner.cpp:37-61): RefMode 0 Zero / 1 Fixed / 2 AdaptiveMean
void write_kernel(BinOut& w, const KernelCfg& k) {
    w.pod<uint32_t>(static_cast<uint32_t>(k.kind));
    w.pod<uint64_t>(k.dim);
    w.pod<double>(k.beta_init);
    w.pod<double>(k.inflation);
    w.pod<uint32_t>(k.adaptive_ref ? 2u : 0u);
    w.vec(Vec{});  // fixed_ref (RefMode::Fixed is not reachable through the C ABI)
    w.pod<uint64_t>(k.n_lag);
    w.pod<double>(k.band_lo);
    w.pod<double>(k.band_hi);
    w.pod<uint64_t>(k.n0);
    w.pod<uint64_t>(k.n_ref_start);
    w.pod<double>(k.beta_adapt_factor);
    w.pod<double>(k.beta_min);
    w.pod<double>(k.beta_max);
    w.pod<uint32_t>(k.adapt_beta ? 1 : 0);
    w.pod<uint32_t>(k.use_explicit_inverse ? 1 : 0);
    w.pod<uint32_t>(0);  // proposal_cov absent
    w.pod<double>(1e-10);
    w.pod<double>(100.0);
    w.pod<double>(1e-4);
}

KernelCfg read_kernel(BinIn& r) {
    KernelCfg k;
    const uint32_t kind = r.pod<uint32_t>();
    require(kind < 4, Err::Io, "corrupt checkpoint: kernel kind");
    k.kind = static_cast<KKind>(kind);
    k.dim = r.pod<uint64_t>();
    k.beta_init = r.pod<double>();
    k.inflation = r.pod<double>();
    const uint32_t ref_mode = r.pod<uint32_t>();
    require(ref_mode == 0 || ref_mode == 2, Err::Io, "checkpoint uses a fixed reference point (unsupported)");
    k.adaptive_ref = ref_mode == 2;
    r.vec();
    k.n_lag = r.pod<uint64_t>();
    k.band_lo = r.pod<double>();
    k.band_hi = r.pod<double>();
    k.n0 = r.pod<uint64_t>();
    k.n_ref_start = r.pod<uint64_t>();
    k.beta_adapt_factor = r.pod<double>();
    k.beta_min = r.pod<double>();
    k.beta_max = r.pod<double>();
    k.adapt_beta = r.pod<uint32_t>() != 0;
    k.use_explicit_inverse = r.pod<uint32_t>() != 0;
    require(r.pod<uint32_t>() == 0, Err::Io, "checkpoint carries a proposal covariance (unsupported)");
    const double e0 = r.pod<double>(), g = r.pod<double>(), em = r.pod<double>();
    require(e0 == 1e-10 && g == 100.0 && em == 1e-4, Err::Io, "checkpoint uses a non-default jitter ladder");
    return k;
}

void write_acc(BinOut& w, size_t d, uint64_t count, const Vec& mean, const Mat& second) {
    w.pod<uint64_t>(d);
    w.pod<uint64_t>(count);
    w.vec(mean);
    w.mat(second);
}

// lower-triangle device rows (ld stride) -> full symmetric host matrix
Mat mirror_lower(const double* h, int d, int64_t ld) {
    Mat m(d, d);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j <= i; ++j) m(i, j) = m(j, i) = h[(size_t)i * ld + j];
    return m;
}

}  // namespace

// One product of device matrices (d x d, row stride ld) on the engine stream, for the
// conversions between the whitened engine state and the checkpoint's x-space fields:
// out = A B (A K-major rows; B rows K-major when bk, else B[k][n]); lower part only if tri.
void Engine::dev_gemm(const double* A, const double* B, bool bk, double* out, bool tri) {
    const double* h[3] = {A, B, out};
    DGB_CUDA(cudaMemcpy(ptr_gen_, h, sizeof(h), cudaMemcpyHostToDevice));
    GemmBatch g{};
    g.A = (const double* const*)ptr_gen_;
    g.B = (const double* const*)(ptr_gen_ + 1);
    g.C = ptr_gen_ + 2;
    g.lda = g.ldb = g.ldc = ld_;
    g.M = g.N = g.K = d_;
    g.alpha = 1.0;
    g.tri_c_lower = tri ? 1 : 0;
    gemm_f64(g, 1, true, bk, stream_);
    DGB_CUDA(cudaStreamSynchronize(stream_));
}

// out (lower) = M sym(S) M^T, S given by its lower triangle (M = G: x -> whitened; M = G^-1:
// whitened -> x); Sfull_ / Stmp_ are the scratch, out may be Sfull_ (not Stmp_)
void Engine::congruence(const double* S, const double* M, double* out) {
    launch_mirror_lower(S, Sfull_, d_, ld_, stream_);
    dev_gemm(Sfull_, M, true, Stmp_, false);  // Sfull M^T (B(k, n) = M[n][k])
    dev_gemm(M, Stmp_, false, out, true);     // M (Sfull M^T), lower
}

void Engine::save_checkpoint(double wall) {
    DGB_CUDA(cudaDeviceSynchronize());
    const int C = C_;
    auto fetch_d = [&](const double* src, size_t n) {
        std::vector<double> v(n);
        DGB_CUDA(cudaMemcpy(v.data(), src, n * 8, cudaMemcpyDeviceToHost));
        return v;
    };
    const auto x = fetch_d(x_, (size_t)C * ld_), xr = fetch_d(xr_, (size_t)C * ld_), y = fetch_d(y_, (size_t)C * ld_);
    const auto lp = fetch_d(logpi_, C), qd = fetch_d(quad_, C), bt = fetch_d(beta_, C);
    // the batch accumulator's x-space mean (the whitened engine keeps it beside its z mean)
    const auto mean = fetch_d(mean_x_, (size_t)C * ld_), cm = fetch_d(cmean_, (size_t)C * ld_);
    const auto sg = fetch_d(Sg_, mat_), mg = fetch_d(mg_, ld_);
    std::vector<uint64_t> uc(C);
    DGB_CUDA(cudaMemcpy(uc.data(), uctr_, C * 8, cudaMemcpyDeviceToHost));
    std::vector<double*> lptr(C);
    DGB_CUDA(cudaMemcpy(lptr.data(), Lp_, C * sizeof(double*), cudaMemcpyDeviceToHost));

    // this rank's chain records (rank order = global chain order under the block sharding)
    // and its part of the B200 extension, in memory; rank 0 writes the file
    BinOut rec, ext;
    const uint64_t nctr = nctr_;
    for (int c = 0; c < C; ++c) {
        rec.vec(Vec(x.begin() + (size_t)c * ld_, x.begin() + (size_t)c * ld_ + d_));
        rec.pod<double>(lp[c]);
        rec.pod<double>(k_.pcn_form() ? qd[c] : 0.0);
        rec.pod<double>(bt[c]);
        rec.pod<uint64_t>(n_);
        rec.pod<uint64_t>(0);  // n_accepted: reset at every lag boundary
        // a lower factor as the reference's full square (zero upper part), row by row
        auto write_lower = [&](const std::vector<double>& m) {
            rec.pod<uint64_t>(d_);
            std::vector<double> row(d_);
            for (int i = 0; i < d_; ++i) {
                for (int j = 0; j < d_; ++j) row[j] = j <= i ? m[(size_t)i * ld_ + j] : 0.0;
                rec.raw(row.data(), row.size() * 8);
            }
        };
        // x-space factor L = G^-1 L_z (the engine factors in whitened space)
        dev_gemm(Ginv_, lptr[c], false, Stmp_, true);
        write_lower(fetch_d(Stmp_, (size_t)d_ * ld_));
        if (Xinv_) {  // factor_inv (runner.cpp:444-445): L^-1 = L_z^-1 G
            rec.pod<uint32_t>(1);
            dev_gemm(Xinv_ + (size_t)c * mat_, G_, false, Stmp_, true);
            write_lower(fetch_d(Stmp_, (size_t)d_ * ld_));
        } else {
            rec.pod<uint32_t>(0);
        }
        rec.vec(k_.adaptive_ref ? Vec(xr.begin() + (size_t)c * ld_, xr.begin() + (size_t)c * ld_ + d_) : Vec(d_, 0.0));
        rec.pod<uint64_t>(nctr);
        rec.pod<uint64_t>(uc[c]);
        // batch accumulator (empty at a batch boundary unless resumed mid-batch)
        Mat sx(d_, d_);
        if (cnt_local_ > 0) {  // the whitened second moments in x-space: G^-1 S_z G^-T
            congruence(S_ + (size_t)c * mat_, Ginv_, Sfull_);
            sx = mirror_lower(fetch_d(Sfull_, mat_).data(), d_, ld_);
        }
        write_acc(rec, d_, cnt_local_, Vec(mean.begin() + (size_t)c * ld_, mean.begin() + (size_t)c * ld_ + d_), sx);
        // cumulative accumulator
        Mat cs(d_, d_);
        if (cS_) {
            congruence(cS_ + (size_t)c * mat_, Ginv_, Sfull_);
            cs = mirror_lower(fetch_d(Sfull_, mat_).data(), d_, ld_);
        }
        write_acc(rec, d_, cum_cnt_, Vec(cm.begin() + (size_t)c * ld_, cm.begin() + (size_t)c * ld_ + d_), cs);
        rec.vec(beta_hist_[c]);
        rec.vec(acc_hist_[c]);
        rec.pod<uint64_t>(fnames_.size());
        for (size_t f = 0; f < fnames_.size(); ++f) rec.vec(traces_[c][f]);
    }
    for (int c = 0; c < C; ++c) ext.vec(Vec(y.begin() + (size_t)c * ld_, y.begin() + (size_t)c * ld_ + d_));
    BinOut ext2;
    {
        auto raw_dev = [&](const double* src, size_t n) {
            const auto v = fetch_d(src, n);
            ext2.raw(v.data(), n * 8);
        };
        for (int c = 0; c < C; ++c) {
            raw_dev(lptr[c], (size_t)mat_);
            if (Xinv_) raw_dev(Xinv_ + (size_t)c * mat_, (size_t)mat_);
            raw_dev(S_ + (size_t)c * mat_, (size_t)mat_);
            if (cS_) raw_dev(cS_ + (size_t)c * mat_, (size_t)mat_);
            raw_dev(mean_ + (size_t)c * ld_, (size_t)ld_);
            raw_dev(diag_x_ + (size_t)c * ld_, (size_t)ld_);
            raw_dev(cdiag_ + (size_t)c * ld_, (size_t)ld_);
        }
    }
    std::vector<char> recs = std::move(rec.mem), exts = std::move(ext.mem), ext2s = std::move(ext2.mem);
    if (comm_) {  // a sharded run: every rank's records to rank 0
        auto all_r = comm_->gather_bytes(recs, stream_);
        auto all_e = comm_->gather_bytes(exts, stream_);
        auto all_e2 = comm_->gather_bytes(ext2s, stream_);
        if (rank_ != 0) return;
        for (int k = 1; k < world_; ++k) {
            recs.insert(recs.end(), all_r[k].begin(), all_r[k].end());
            exts.insert(exts.end(), all_e[k].begin(), all_e[k].end());
            ext2s.insert(ext2s.end(), all_e2[k].begin(), all_e2[k].end());
        }
    }
    BinOut w(cfg_.checkpoint_path);
    w.raw(kCkptMagic, 8);
    w.pod<uint32_t>(kVersion);
    w.pod<uint32_t>(kEndian);
    write_target_blob(w, tgt_);
    write_kernel(w, k_);
    w.pod<uint64_t>(cfg_.chains);
    w.pod<uint64_t>(cfg_.intervals_per_batch);
    w.pod<uint64_t>(cfg_.max_batches);
    write_opt(w, cfg_.cov_tol);
    write_opt(w, cfg_.mean_tol);
    write_opt(w, cfg_.psrf_tol);
    w.pod<uint32_t>(cfg_.max_samples ? 1 : 0);
    w.pod<uint64_t>(cfg_.max_samples.value_or(0));
    write_opt(w, cfg_.max_wall_seconds);
    w.pod<double>(cfg_.init_dispersion);
    w.pod<uint64_t>(cfg_.master_seed);
    w.pod<uint32_t>(cfg_.record_traces ? 1 : 0);
    w.pod<uint64_t>(cfg_.trace_thin);
    w.pod<uint32_t>(cfg_.trace_eigen_projections ? 1 : 0);
    w.pod<uint64_t>(0);  // no extra eigen trace indices through the C ABI
    w.str(cfg_.checkpoint_path);
    w.pod<uint64_t>(cfg_.threads);

    w.pod<uint64_t>(batches_done_);
    w.pod<uint64_t>(batches_done_);  // global.batches: one merge per finished batch
    w.pod<uint64_t>(cnt_g_);
    w.vec(Vec(mg.begin(), mg.begin() + d_));
    w.mat(mirror_lower(sg.data(), d_, ld_));
    w.pod<double>(wall);
    w.vec(batch_seconds_);
    w.vec(cov_hist_);
    w.vec(mean_hist_);
    w.vec(psrf_hist_);

    w.pod<uint64_t>((uint64_t)P_);
    w.raw(recs.data(), recs.size());
    // B200 extension: the recursively carried y
    w.raw(kExtMagic, 8);
    w.raw(exts.data(), exts.size());
    w.raw(kExt2Magic, 8);
    {
        const auto sgz = fetch_d(Sgz_, (size_t)mat_), mgz = fetch_d(mgz_, (size_t)ld_);
        w.raw(sgz.data(), sgz.size() * 8);
        w.raw(mgz.data(), mgz.size() * 8);
    }
    w.raw(ext2s.data(), ext2s.size());
    w.close();
}

void Engine::read_checkpoint_header(BinIn& r, HostTarget& t, RunCfg& cfg) {
    char magic[8];
    r.raw(magic, 8);
    require(std::memcmp(magic, kCkptMagic, 8) == 0, Err::Io, "not a checkpoint file");
    require(r.pod<uint32_t>() == kVersion, Err::Io, "unsupported checkpoint version");
    require(r.pod<uint32_t>() == kEndian, Err::Io, "endianness mismatch in checkpoint");
    t = read_target_blob(r);
    cfg.kernel = read_kernel(r);
    cfg.chains = r.pod<uint64_t>();
    cfg.intervals_per_batch = r.pod<uint64_t>();
    cfg.max_batches = r.pod<uint64_t>();
    cfg.cov_tol = read_opt(r);
    cfg.mean_tol = read_opt(r);
    cfg.psrf_tol = read_opt(r);
    const bool has_ms = r.pod<uint32_t>() != 0;
    const uint64_t ms = r.pod<uint64_t>();
    if (has_ms) cfg.max_samples = ms;
    cfg.max_wall_seconds = read_opt(r);
    cfg.init_dispersion = r.pod<double>();
    cfg.master_seed = r.pod<uint64_t>();
    cfg.record_traces = r.pod<uint32_t>() != 0;
    cfg.trace_thin = r.pod<uint64_t>();
    cfg.trace_eigen_projections = r.pod<uint32_t>() != 0;
    const uint64_t extra = r.pod<uint64_t>();
    require(extra == 0, Err::Io, "checkpoint traces extra eigen directions (unsupported)");
    cfg.checkpoint_path = r.str();
    cfg.threads = r.pod<uint64_t>();
}

void Engine::restore(BinIn& r) {  // proj/src/runner.cpp:164-206
    // a sharded engine (rank r of N) reads every chain's record and keeps its own
    // [c0, c0 + C); the shared state (global moments, histories) is the same for every rank
    const int C = C_;
    batches_done_ = r.pod<uint64_t>();
    r.pod<uint64_t>();  // global.batches
    cnt_g_ = r.pod<uint64_t>();
    const Vec gmean = r.vec();
    const Mat gsec = r.mat();
    require(gmean.size() == (size_t)d_ && gsec.rows == (size_t)d_, Err::Io, "corrupt checkpoint: global moments");
    wall_accum_ = r.pod<double>();
    batch_seconds_ = r.vec();
    cov_hist_ = r.vec();
    mean_hist_ = r.vec();
    psrf_hist_ = r.vec();
    require(r.pod<uint64_t>() == (uint64_t)P_, Err::Io, "checkpoint chain count mismatch");

    auto put = [&](double* dst, const double* src, size_t n) {
        DGB_CUDA(cudaMemcpy(dst, src, n * 8, cudaMemcpyHostToDevice));
    };
    auto put_lower = [&](double* dst, const Mat& m) {  // full host -> lower device rows (upper zero)
        std::vector<double> buf((size_t)d_ * ld_, 0.0);
        for (int i = 0; i < d_; ++i)
            for (int j = 0; j <= i; ++j) buf[(size_t)i * ld_ + j] = m(i, j);
        put(dst, buf.data(), buf.size());
    };
    {
        std::vector<double> m(ld_, 0.0);
        std::copy(gmean.begin(), gmean.end(), m.begin());
        put(mg_, m.data(), ld_);
        put_lower(Sg_, gsec);
        // the whitened snapshot: Sgz = G Sg G^T, mgz = G mg
        congruence(Sg_, G_, Sgz_);
        launch_gemv_rows(G_, ld_, d_, d_, mg_, mgz_, ld_, 1, stream_);
    }
    std::vector<double> lp(C), qd(C), bt(C);
    std::vector<uint64_t> uc(C);
    uint64_t nctr = 0, n = 0, cnt_local = 0, cum = 0;
    std::vector<double*> lptr(C);
    DGB_CUDA(cudaMemcpy(lptr.data(), Lp_, C * sizeof(double*), cudaMemcpyDeviceToHost));
    bool all_identity = true, need_inverse = false;
    for (int pg = 0; pg < P_; ++pg) {
        const bool mine = pg >= c0_ && pg < c0_ + C;
        const int c = mine ? pg - c0_ : 0;
        std::vector<double> row(ld_, 0.0);
        const Vec x = r.vec();
        require(x.size() == (size_t)d_, Err::Io, "corrupt checkpoint: state");
        std::copy(x.begin(), x.end(), row.begin());
        if (mine) put(x_ + (size_t)c * ld_, row.data(), ld_);
        const double lpv = r.pod<double>(), qdv = r.pod<double>(), btv = r.pod<double>();
        if (mine) {
            lp[c] = lpv;
            qd[c] = qdv;
            bt[c] = btv;
        }
        const uint64_t nc = r.pod<uint64_t>();
        require(pg == 0 || nc == n, Err::Io, "chains at different iteration counts");
        n = nc;
        r.pod<uint64_t>();  // n_accepted
        const uint64_t dim = r.pod<uint64_t>();
        require(dim == (uint64_t)d_, Err::Io, "corrupt checkpoint: factor");
        if (mine) {
            Mat L(d_, d_);
            r.raw(L.a.data(), L.a.size() * 8);
            for (int i = 0; i < d_ && all_identity; ++i)
                for (int j = 0; j <= i; ++j)
                    if (L(i, j) != (i == j ? 1.0 : 0.0)) {
                        all_identity = false;
                        break;
                    }
            put_lower(lptr[c], L);
            dev_gemm(G_, lptr[c], false, Stmp_, true);  // whitened factor L_z = G L
            DGB_CUDA(cudaMemcpyAsync(lptr[c], Stmp_, (size_t)mat_ * 8, cudaMemcpyDeviceToDevice, stream_));
        } else {
            r.skip((size_t)d_ * d_ * 8);
        }
        if (r.pod<uint32_t>() != 0) {  // factor_inv (runner.cpp:186)
            require(r.pod<uint64_t>() == (uint64_t)d_, Err::Io, "corrupt checkpoint: inverse factor");
            if (mine) {
                Mat X(d_, d_);
                r.raw(X.a.data(), X.a.size() * 8);
                if (Xinv_) {  // L_z^-1 = L^-1 G^-1
                    put_lower(Xinv_ + (size_t)c * mat_, X);
                    dev_gemm(Xinv_ + (size_t)c * mat_, Ginv_, false, Stmp_, true);
                    DGB_CUDA(cudaMemcpyAsync(Xinv_ + (size_t)c * mat_, Stmp_, (size_t)mat_ * 8, cudaMemcpyDeviceToDevice,
                                             stream_));
                }
            } else {
                r.skip((size_t)d_ * d_ * 8);
            }
        } else if (Xinv_) {  // a file without the inverse: recomputed below from the factor
            need_inverse = true;
        }
        const Vec xr = r.vec();
        std::fill(row.begin(), row.end(), 0.0);
        std::copy(xr.begin(), xr.end(), row.begin());
        if (mine) put(xr_ + (size_t)c * ld_, row.data(), ld_);
        const uint64_t nc_ctr = r.pod<uint64_t>();
        require(pg == 0 || nc_ctr == nctr, Err::Io, "chains at different noise-stream positions");
        nctr = nc_ctr;
        const uint64_t ucv = r.pod<uint64_t>();
        if (mine) uc[c] = ucv;
        for (int which = 0; which < 2; ++which) {  // batch, then cumulative accumulator
            r.pod<uint64_t>();
            const uint64_t cnt = r.pod<uint64_t>();
            const Vec m = r.vec();
            if (!mine) {
                r.skip_mat();
                if (which == 0) cnt_local = cnt;
                else cum = cnt;
                continue;
            }
            const Mat s = r.mat();
            std::fill(row.begin(), row.end(), 0.0);
            std::copy(m.begin(), m.end(), row.begin());
            std::vector<double> dg(ld_, 0.0);
            for (int i = 0; i < d_; ++i) dg[i] = s(i, i);
            if (which == 0) {  // x-space mean and raw diagonal; whitened S_z = G S G^T
                cnt_local = cnt;
                put(mean_x_ + (size_t)c * ld_, row.data(), ld_);
                put(diag_x_ + (size_t)c * ld_, dg.data(), ld_);
                put_lower(S_ + (size_t)c * mat_, s);
                congruence(S_ + (size_t)c * mat_, G_, S_ + (size_t)c * mat_);
            } else {
                cum = cnt;
                put(cmean_ + (size_t)c * ld_, row.data(), ld_);
                put(cdiag_ + (size_t)c * ld_, dg.data(), ld_);
                if (cS_) {
                    put_lower(cS_ + (size_t)c * mat_, s);
                    congruence(cS_ + (size_t)c * mat_, G_, cS_ + (size_t)c * mat_);
                }
            }
        }
        Vec bh = r.vec(), ah = r.vec();
        const uint64_t nf = r.pod<uint64_t>();
        require(nf == fnames_.size(), Err::Io, "checkpoint functional count mismatch");
        std::vector<Vec> tr(nf);
        for (size_t f = 0; f < nf; ++f) tr[f] = r.vec();
        if (mine) {
            beta_hist_[c] = std::move(bh);
            acc_hist_[c] = std::move(ah);
            for (size_t f = 0; f < nf; ++f) traces_[c][f] = std::move(tr[f]);
        }
    }
    put(logpi_, lp.data(), C);
    put(quad_, qd.data(), C);
    put(beta_, bt.data(), C);
    DGB_CUDA(cudaMemcpy(uctr_, uc.data(), C * 8, cudaMemcpyHostToDevice));
    n_ = n;
    nctr_ = nctr;
    cnt_local_ = cnt_local;
    cum_cnt_ = cum;
    identity_ = all_identity;

    // derived device state: the whitened batch mean, G x, G x_ref, X_z = L_z^-1 (a file
    // without it) and y = L^-1 (x - x_ref) = L_z^-1 (z - z_ref)
    launch_gemv_rows(G_, ld_, d_, d_, mean_x_, mean_, ld_, C, stream_);
    if (need_inverse) trtri_batched(Lp_, Xinvp_, Tinvp_, ld_, d_, C, nullptr, stream_);
    refresh_g(x_, g_, C, stream_);
    if (k_.adaptive_ref) refresh_g(xr_, gr_, C, stream_);
    DGB_CUDA(cudaStreamSynchronize(stream_));
    bool have_y = false;
    if (!r.at_end()) {
        char magic[8];
        r.raw(magic, 8);
        if (std::memcmp(magic, kExtMagic, 8) == 0) {
            for (int pg = 0; pg < P_; ++pg) {
                const Vec y = r.vec();
                if (pg < c0_ || pg >= c0_ + C) continue;
                std::vector<double> row(ld_, 0.0);
                std::copy(y.begin(), y.end(), row.begin());
                put(y_ + (size_t)(pg - c0_) * ld_, row.data(), ld_);
            }
            have_y = true;
            if (!r.at_end()) {
                r.raw(magic, 8);
                if (std::memcmp(magic, kExt2Magic, 8) == 0) {  // this engine's exact whitened state
                    std::vector<double> buf((size_t)mat_);
                    auto get = [&](double* dst, size_t n, bool keep) {
                        if (!keep) {
                            r.skip(n * 8);
                            return;
                        }
                        r.raw(buf.data(), n * 8);
                        put(dst, buf.data(), n);
                    };
                    get(Sgz_, (size_t)mat_, true);
                    get(mgz_, (size_t)ld_, true);
                    for (int pg = 0; pg < P_; ++pg) {
                        const bool mine = pg >= c0_ && pg < c0_ + C;
                        const int c = mine ? pg - c0_ : 0;
                        get(lptr[c], (size_t)mat_, mine);
                        if (Xinv_) get(Xinv_ + (size_t)c * mat_, (size_t)mat_, mine);
                        get(S_ + (size_t)c * mat_, (size_t)mat_, mine);
                        if (cS_) get(cS_ + (size_t)c * mat_, (size_t)mat_, mine);
                        get(mean_ + (size_t)c * ld_, (size_t)ld_, mine);
                        get(diag_x_ + (size_t)c * ld_, (size_t)ld_, mine);
                        get(cdiag_ + (size_t)c * ld_, (size_t)ld_, mine);
                    }
                }
            }
        }
    }
    if (k_.pcn_form() && !have_y) {
        // reference-written checkpoint: solve y; keep the saved quad (the reference's value)
        const double infl = k_.noise_infl();
        launch_trsv(Lp_, ld_, g_, k_.adaptive_ref ? gr_ : nullptr, ldg_, y_, ld_, qtmp_, C, d_, 0.5 / (infl * infl),
                    nullptr, stream_);
    }
    DGB_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::override_stop(const RunCfg& c) {
    cfg_.cov_tol = c.cov_tol;
    cfg_.mean_tol = c.mean_tol;
    cfg_.psrf_tol = c.psrf_tol;
    cfg_.max_samples = c.max_samples;
    cfg_.max_wall_seconds = c.max_wall_seconds;
    validate_run_cfg(cfg_, tgt_);
}

}  // namespace dgb
