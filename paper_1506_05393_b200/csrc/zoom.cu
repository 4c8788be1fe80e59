// zoom.cu -- K5 host orchestration: run_quantify (quantify_impl per voxel,
// reference proj/src/zoom.cpp:416-523; the device code is zoom_dev.cuh, the
// kernel variants live in zoom_k_*.cu).
#include "zoom_dev.cuh"

namespace mrfg {

void run_quantify(Ctx& c, const mrfg_grid& lat, const mrfg_zoom_config& cfg, const double* d_fps,
                  int64_t nvox, const int64_t* h_bounds, const double* h_init, mrfg_quant* d_out,
                  int64_t nrows, const int64_t* h_row_start, const int64_t* h_vox_list, const float* d_dict,
                  int64_t dict_entries, mrfg_stage* d_trace, int* d_trace_len, const int* d_vox_ib,
                  Ctx* const* sched, int nsched) {
    for (const mrfg_axis* ax : {&lat.t1_ms, &lat.t2_ms, &lat.df_hz})
        MRFG_REQUIRE(ax->count > 0 && ax->count < (int64_t(1) << 21), MRFG_E_INVALID,
                     "objective: lattice axis empty or too fine");  // zoom.cpp:46-48
    MRFG_REQUIRE(cfg.smooth_k == 0 || cfg.smooth_k == 3 || cfg.smooth_k == 5, MRFG_E_INVALID,
                 "smooth: kernel must be 3 or 5");  // fingerprint.cpp:123
    MRFG_REQUIRE(cfg.n2d >= 0 && cfg.n2d <= 8 && cfg.n1d >= 0 && cfg.n1d <= 8, MRFG_E_INVALID,
                 "quantify: at most 8 zoom steps per stage");
    MRFG_REQUIRE(!grid_explicit(lat), MRFG_E_INVALID,
                 "quantify: the search lattice must be evenly spaced (explicit axis values are for "
                 "generate / scan_grid / cc_map)");
    const GridTables& t = ensure_tables(c, lat, true);
    ZParams P{};
    P.rf = c.rf64_d.as<double>();
    P.e1d = t.e1d.as<double>();
    P.e2d = t.e2d.as<double>();
    P.phd = t.phd.as<double>();
    P.su = t.stepu.as<float4>();
    // x-axis screening rows (FP32 screening only: the exact FP64 walk keeps
    // the full matrices, the MUFU and smoothing screens the StepU rows);
    // MRFG_ZOOM_XR=0 forces the general rows
    {
        const char* xe = std::getenv("MRFG_ZOOM_XR");
        const char* sm = std::getenv("MRFG_ZOOM_SCREEN");
        P.xr = c.rf_xaxis && t.stepx.p && cfg.smooth_k == 0 && !(sm && std::string(sm) == "mufu") &&
               !(xe && std::atoi(xe) == 0);
        P.sut = P.xr ? t.stepx.as<float4>() : P.su;
        P.sus = P.xr ? 2 : 4;
    }
    P.e1f = t.e1f.as<float4>();
    P.e2f = t.e2f.as<float2>();
    P.phf = t.phf.as<float4>();
    P.inv0[0] = c.inv64[2];
    P.inv0[1] = c.inv64[5];
    P.inv0[2] = c.inv64[8];
    P.n = static_cast<int>(c.n);
    P.L = {lat.t1_ms.count, lat.t2_ms.count, lat.df_hz.count};
    P.t1_min = lat.t1_ms.min;
    P.t1_step = lat.t1_ms.step;
    P.t2_min = lat.t2_ms.min;
    P.t2_step = lat.t2_ms.step;
    P.df_min = lat.df_hz.min;
    P.df_step = lat.df_hz.step;
    MRFG_REQUIRE(cfg.dict_mode >= 0 && cfg.dict_mode <= 2, MRFG_E_INVALID, "quantify: bad dictionary mode");
    P.dict_mode = cfg.dict_mode;
    if (d_dict) {  // zoom.cpp:101-113: the df slab (entry idf) or the full lattice dictionary
        MRFG_REQUIRE(cfg.dict_mode != 0, MRFG_E_INVALID, "quantify: dictionary payload without a dictionary mode");
        const int64_t need = cfg.dict_mode == 2 ? grid_total(lat) : lat.df_hz.count;
        MRFG_REQUIRE(dict_entries == need, MRFG_E_INVALID, "objective: dictionary does not match the lattice");
    }
    P.dict = reinterpret_cast<const float2*>(d_dict);
    P.trace = d_trace;
    P.trace_len = d_trace_len;
    P.smooth_k = cfg.smooth_k;
    if (cfg.smooth_k) {  // fingerprint.cpp:125-129, host libm
        const double sigma = cfg.smooth_k == 3 ? 0.85 : 1.0;
        const int h = cfg.smooth_k / 2;
        for (int j = -h; j <= h; ++j) {
            P.sw[j + h] = std::exp(-0.5 * j * j / (sigma * sigma));
            P.swf[j + h] = static_cast<float>(P.sw[j + h]);
        }
    }
    P.metric = cfg.metric;
    P.final_metric = cfg.final_metric;
    P.need_euc = cfg.metric == MRFG_METRIC_EUCLIDEAN || cfg.final_metric == MRFG_METRIC_EUCLIDEAN;
    // zoom.cpp:454-463
    const double dfs = lat.df_hz.step;
    P.df_coarse = step_units(cfg.df_coarse_hz, dfs);
    P.df_refine = step_units(cfg.df_refine_hz, dfs);
    P.df_window_half = step_units(cfg.df_window_hz / 2, dfs);
    P.omega = step_units(cfg.omega_hz, dfs);
    P.plateau_eps = cfg.plateau_eps;
    P.heavy_cc = cfg.metric == MRFG_METRIC_CC ? cfg.heavy_noise_cc : -1e300;
    P.fb_coarse = step_units(cfg.fallback_coarse_hz, dfs);
    P.fb_window_half = step_units(cfg.fallback_window_hz / 2, dfs);
    P.n2d = cfg.n2d;
    P.n1d = cfg.n1d;
    for (int k = 0; k < cfg.n2d; ++k) {
        P.s2d1[k] = step_units(cfg.t1t2_2d_steps_ms[k], lat.t1_ms.step);
        P.s2d2[k] = step_units(cfg.t1t2_2d_steps_ms[k], lat.t2_ms.step);
    }
    for (int k = 0; k < cfg.n1d; ++k) {
        P.s1d1[k] = step_units(cfg.t1t2_1d_steps_ms[k], lat.t1_ms.step);
        P.s1d2[k] = step_units(cfg.t1t2_1d_steps_ms[k], lat.t2_ms.step);
    }
    P.f2d1 = step_units(cfg.final_2d_step_ms, lat.t1_ms.step);
    P.f2d2 = step_units(cfg.final_2d_step_ms, lat.t2_ms.step);
    {
        const char* e1 = std::getenv("MRFG_ZOOM_SPEC1D");
        const char* e2 = std::getenv("MRFG_ZOOM_SPEC2D");
        // speculation widths, re-measured after the packed screening step
        // (ms, config 2 / config 4): 1-D/2-D 8/1: 17.4 / 66.6-67.1;
        // 16/2: 19.1-19.3 / 67.6-68.3.  The helper-warp (rows) kernel keeps 16/2.
        P.spec1d = e1 ? std::max(1, std::atoi(e1)) : 8;
        P.spec2d = e2 ? std::max(1, std::atoi(e2)) : 1;
        const char* c1 = std::getenv("MRFG_ZOOM_SPEC1D_CTA");
        const char* c2 = std::getenv("MRFG_ZOOM_SPEC2D_CTA");
        P.spec1d_cta = c1 ? std::max(1, std::atoi(c1)) : (e1 ? P.spec1d : 16);
        P.spec2d_cta = c2 ? std::max(1, std::atoi(c2)) : (e2 ? P.spec2d : 2);
        const char* sm = std::getenv("MRFG_ZOOM_SCREEN");
        const std::string smode = sm ? sm : "";
        // (a third variant -- E1/E2 by MUFU.EX2, phasor rows streamed --
        // measured 83 vs 65 ms on config 4 with 8x the screening error: dropped)
        P.screen_mode = smode == "mufu" ? 1 : 0;
        const char* ee = std::getenv("MRFG_ZOOM_EPS");
        P.eps = ee ? std::atof(ee) : 1e-5;
        // |sqrt(a) - sqrt(b)| <= sqrt(|a - b|), |d dd| <= 2 eps
        P.eps_euc = P.eps < 0 ? P.eps : std::sqrt(2.0 * P.eps) * 1.01 + 1e-12;
    }
    const bool want_stats = std::getenv("MRFG_ZOOM_STATS") != nullptr;
    const char* vs_file = std::getenv("MRFG_ZOOM_STATS_FILE");
    P.init1 = snap_index(cfg.init_t1_ms, lat.t1_ms);
    P.init2 = snap_index(cfg.init_t2_ms, lat.t2_ms);
    P.fps = d_fps;
    const unsigned int cap = 8192;
    P.cap_mask = cap - 1;
    P.nvox = nvox;
    // persistent warps: as many as are co-resident (at most one per voxel)
    // block size: 8 warps (one StepU copy per SM, so L1 keeps room for the
    // per-lane table streams) or 4 warps (MRFG_ZOOM_BS=128)
    const char* bs_env = std::getenv("MRFG_ZOOM_BS");
    const int bs_req = bs_env ? std::atoi(bs_env) : 256;
    const int bs = bs_req == 128 ? 128 : (bs_req == 512 ? 512 : 256);
    // register budget: minimum resident blocks per SM (128 threads: 1, 4 or 6;
    // 256 threads: 1 or 2)
    const char* mb_env = std::getenv("MRFG_ZOOM_MINB");
    const int minb = mb_env ? std::atoi(mb_env) : 1;
    const bool rows = nrows > 0;
    // rows mode: one warp per block (a row's voxels are a latency chain: one
    // row per SM)
    // rows mode: one row per block of row_w warps (warp 0 decides, all warps
    // evaluate; MRFG_ZOOM_ROWW = 1, 4 or 8)
    const char* rw_env = std::getenv("MRFG_ZOOM_ROWW");
    const int row_w = rw_env ? (std::atoi(rw_env) >= 8 ? 8 : (std::atoi(rw_env) >= 4 ? 4 : 1)) : 8;
    const int variant = rows ? (row_w == 8 ? kZoomRows256 : (row_w == 4 ? kZoomRows128 : kZoomRows32))
                        : bs == 512 ? kZoom512x1
                        : bs == 256 ? (minb >= 2 ? kZoom256x2 : kZoom256x1)
                                    : (minb >= 6 ? kZoom128x6 : (minb >= 4 ? kZoom128x4 : kZoom128x1));
    auto run_variant = [&](bool launch, unsigned grid, int block, size_t sm, int* occ) {
        const void* pp = &P;
        if (!zoom_tu_main(variant, pp, launch, grid, block, sm, c.stream, occ) &&
            !zoom_tu_rows(variant, pp, launch, grid, block, sm, c.stream, occ) &&
            !zoom_tu_var(variant, pp, launch, grid, block, sm, c.stream, occ))
            throw Error{MRFG_E_RUNTIME, "quantify: kernel variant not built"};
    };
    const int bsk = rows ? 32 * row_w : bs;
    // shared staging: StepU rows (64 B/step) + one FP32 query per warp (8 B/step)
    const size_t row_bytes = sizeof(float4) * P.sus;  // staged screening step row
    size_t smem = rows ? row_bytes * c.n + sizeof(float2) * c.n + sizeof(ZItem) * kQCap + 16
                       : (row_bytes + sizeof(float2) * (bsk / 32)) * c.n;
    const char* st_env = std::getenv("MRFG_ZOOM_SMEM");
    P.smem_stage = smem <= 200 * 1024 && !(st_env && std::atoi(st_env) == 0) && !d_vox_ib ? 1 : 0;
    // CTA mode (the slice kernels): small rounds screened parallel in time,
    // one point per warp (x-axis rows; not with smoothing, MUFU screening or
    // the all-FP64 mode); MRFG_ZOOM_PIT=0 disables it
    {
        const char* pe = std::getenv("MRFG_ZOOM_PIT");
        P.pit = P.xr && P.eps >= 0 && P.screen_mode == 0 && !P.smooth_k && !(pe && std::atoi(pe) == 0) ? 1 : 0;
    }
    P.vox_ib = d_vox_ib;
    if (d_vox_ib) {
        MRFG_REQUIRE(!rows && nsched > 0 && nsched <= 16, MRFG_E_INVALID, "quantify: 1 to 16 schedules per launch");
        for (int k = 0; k < nsched; ++k) {
            Ctx& s = *sched[k];
            MRFG_REQUIRE(s.n == c.n && s.device == c.device && s.rf_xaxis == c.rf_xaxis, MRFG_E_INVALID,
                         "quantify: schedules differ in length, device or RF axis");
            const GridTables& tk = ensure_tables(s, lat, true);
            if (&s != &c) MRFG_CUDA(cudaStreamSynchronize(s.stream));  // its table uploads
            P.rf_b[k] = s.rf64_d.as<double>();
            P.sut_b[k] = P.xr ? tk.stepx.as<float4>() : tk.stepu.as<float4>();
        }
    }
    // rows mode keeps its shared layout (the helper-warp queue follows the
    // staged rows) whether or not the kernel reads the staged copies
    MRFG_REQUIRE(!rows || smem <= 200 * 1024, MRFG_E_INVALID,
                 "quantify_slice: schedule too long for the neighbour-seeded kernel");
    if (!P.smem_stage && !rows) smem = 0;
    int per_sm = 0;
    run_variant(false, 0, bsk, smem, &per_sm);
    const int64_t resident = int64_t(std::max(per_sm, 1)) * c.num_sms * (bsk / 32);
    MRFG_REQUIRE(!rows || nrows * row_w <= resident, MRFG_E_RUNTIME,
                 "quantify_slice: more raster rows than resident blocks");
    const int64_t nwarps = rows ? nrows * row_w : std::min<int64_t>(resident, round_up(nvox, bs / 32));
    // scratch: per-warp queries, fingerprints and memo tables; per-voxel
    // bounds/inits; error flag, stats, work counter
    const size_t qbytes = (sizeof(double) * 2 + sizeof(float) * 2) * c.n * nwarps;
    const size_t fbytes = sizeof(double2) * 32 * c.n * nwarps;
    const size_t tbytes = sizeof(ZSlot) * cap * nwarps;
    const size_t pbytes = sizeof(int) * kPendCap * nwarps;
    const size_t dbytes = sizeof(ZDec) * kDecCap * nwarps;
    const size_t bbytes = h_bounds ? sizeof(long long) * 6 * nvox : 0;
    const size_t rbytes = rows ? sizeof(int64_t) * (nrows + 1 + h_row_start[nrows]) + sizeof(int) * nvox : 0;
    const size_t ibytes = h_init ? sizeof(long long) * 2 * nvox : 0;
    const size_t vbytes = want_stats ? sizeof(long long) * 4 * nvox : 0;
    DevBuf& scratch = c.zoom;
    scratch.ensure(fbytes + qbytes + tbytes + dbytes + pbytes + bbytes + ibytes + rbytes + 256 + vbytes);
    char* base = scratch.as<char>();
    P.fpx = reinterpret_cast<double2*>(base);
    base += fbytes;
    P.q = reinterpret_cast<double*>(base);
    P.q32 = reinterpret_cast<float2*>(base + sizeof(double) * 2 * c.n * nwarps);
    base += qbytes;
    P.tab = reinterpret_cast<ZSlot*>(base);
    base += tbytes;
    P.dec = reinterpret_cast<ZDec*>(base);
    base += dbytes;
    P.pend = reinterpret_cast<int*>(base);
    base += pbytes;
    P.bounds = h_bounds ? reinterpret_cast<long long*>(base) : nullptr;
    base += bbytes;
    P.inits = h_init ? reinterpret_cast<long long*>(base) : nullptr;
    base += ibytes;
    P.nrows = rows ? nrows : 0;
    if (rows) {
        const int64_t m = h_row_start[nrows];
        int64_t* rs = reinterpret_cast<int64_t*>(base);
        int64_t* vl = rs + nrows + 1;
        P.row_start = rs;
        P.vox_list = vl;
        P.done = reinterpret_cast<int*>(vl + m);
        MRFG_CUDA(cudaMemcpyAsync(rs, h_row_start, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice, c.stream));
        MRFG_CUDA(cudaMemcpyAsync(vl, h_vox_list, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c.stream));
        MRFG_CUDA(cudaMemsetAsync(P.done, 0, sizeof(int) * nvox, c.stream));
        P.pw1 = step_units(cfg.prior_window_t1_ms, lat.t1_ms.step);  // zoom.cpp:600-602
        P.pw2 = step_units(cfg.prior_window_t2_ms, lat.t2_ms.step);
        P.pwdf = step_units(cfg.prior_window_df_hz, lat.df_hz.step);
    }
    base += rbytes;
    P.err = reinterpret_cast<int*>(base);
    P.next = reinterpret_cast<unsigned long long*>(base + 64);
    P.stats = want_stats ? reinterpret_cast<unsigned long long*>(base + 128) : nullptr;
    P.vstats = want_stats ? reinterpret_cast<long long*>(base + 256) : nullptr;
    MRFG_CUDA(cudaMemsetAsync(P.next, 0, sizeof(unsigned long long), c.stream));
    MRFG_CUDA(cudaMemsetAsync(P.err, 0, sizeof(int), c.stream));
    if (P.stats) MRFG_CUDA(cudaMemsetAsync(P.stats, 0, 128, c.stream));
    static_assert(sizeof(unsigned long long) * 16 <= 128, "stats block");
    if (h_bounds)
        MRFG_CUDA(cudaMemcpyAsync(const_cast<long long*>(P.bounds), h_bounds, bbytes,
                                  cudaMemcpyHostToDevice, c.stream));
    std::vector<long long> inits;
    if (h_init) {
        inits.resize(2 * nvox);
        for (int64_t k = 0; k < nvox; ++k) {
            inits[2 * k] = snap_index(h_init[2 * k], lat.t1_ms);
            inits[2 * k + 1] = snap_index(h_init[2 * k + 1], lat.t2_ms);
        }
        MRFG_CUDA(cudaMemcpyAsync(const_cast<long long*>(P.inits), inits.data(), ibytes,
                                  cudaMemcpyHostToDevice, c.stream));
    }
    P.out = d_out;
    run_variant(true, static_cast<unsigned>((nwarps + bsk / 32 - 1) / (bsk / 32)), bsk, smem, nullptr);
    int err = 0;
    MRFG_CUDA(cudaMemcpyAsync(&err, P.err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    unsigned long long st[16] = {};
    std::vector<long long> vst(want_stats ? 4 * nvox : 0);
    if (P.stats) {
        MRFG_CUDA(cudaMemcpyAsync(st, P.stats, 128, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaMemcpyAsync(vst.data(), P.vstats, vbytes, cudaMemcpyDeviceToHost, c.stream));
    }
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    if (P.stats)
        std::fprintf(stderr,
                     "[mrfg zoom] voxels %lld fp32 %llu fp64 %llu fp64_rounds %llu near_ties %llu "
                     "cyc/voxel mean %.0f max %llu screen %.0f exact %.0f max|screen-exact| %.3g passes %llu "
                     "audit %llu max|err| %.3g rounds(big) %llu lanes %.1f rounds(small) %llu lanes %.1f\n",
                     static_cast<long long>(nvox), st[0], st[1], st[2], st[3],
                     double(st[4]) / double(nvox), st[5], double(st[6]) / double(nvox),
                     double(st[7]) / double(nvox), [&] {
                         double d;
                         std::memcpy(&d, &st[8], 8);
                         return d;
                     }(), st[9], st[11], [&] {
                         double d;
                         std::memcpy(&d, &st[10], 8);
                         return d;
                     }(), st[12], double(st[13]) / double(st[12] ? st[12] : 1), st[14],
                     double(st[15]) / double(st[14] ? st[14] : 1));
    if (P.stats && vs_file) {
        if (FILE* f = std::fopen(vs_file, "wb")) {
            std::fwrite(vst.data(), sizeof(long long), vst.size(), f);
            std::fclose(f);
        }
    }
    MRFG_REQUIRE(err != 1, MRFG_E_RANGE, "objective: lattice index out of range");
    MRFG_REQUIRE(err != 2, MRFG_E_RUNTIME, "quantify: per-voxel memo table full");
    MRFG_REQUIRE(err != 3, MRFG_E_INVALID, "normalize: zero fingerprint");
}

}  // namespace mrfg
