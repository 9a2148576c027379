// tk_abi_map.cu — the C ABI of the mapping iteration (include/tk_render.h "mapping"): keyframes,
// optimize_step (losses, backward, Adam), statistics, insert_gaussians and prune_map.
#include "tk_abi_internal.cuh"

namespace {

// Grow a device array to new_count elements keeping the first old_count (structural edits).
template <class T>
T* grow_keep(tk_ctx* c, DevBuf& b, int64_t old_count, int64_t new_count, bool zero_tail) {
    const size_t need = static_cast<size_t>(std::max<int64_t>(new_count, 1)) * sizeof(T);
    if (b.bytes < need) {
        DevBuf nb;
        nb.p = pool_alloc(tk::align_bytes(need + need / 8), &nb.bytes);
        if (old_count > 0 && b.p)
            CK(cudaMemcpyAsync(nb.p, b.p, old_count * sizeof(T), cudaMemcpyDeviceToDevice, c->cur));
        CK(cudaStreamSynchronize(c->cur));
        b = std::move(nb);
    }
    if (zero_tail && new_count > old_count)
        CK(cudaMemsetAsync(ptr<T>(b) + old_count, 0, (new_count - old_count) * sizeof(T), c->cur));
    return ptr<T>(b);
}

// Keep the rows flagged in keep (n rows of `width` elements) in order, into a fresh buffer.
template <class T>
void compact_rows(tk_ctx* c, DevBuf& b, int64_t n, int width, int64_t n_keep, const int32_t* keep,
                  const int32_t* pos) {
    if (!b.p || width <= 0) return;
    DevBuf nb;
    ensure<T>(nb, std::max<int64_t>(n_keep, 1) * width);
    if (sizeof(T) == 8)
        tk::launch_compact_f64(reinterpret_cast<const double*>(b.p), static_cast<double*>(nb.p), keep, pos, n, width,
                               c->cur);
    else
        tk::launch_compact_f32(reinterpret_cast<const float*>(b.p), static_cast<float*>(nb.p), keep, pos, n, width,
                               c->cur);
    CK_LAUNCH(c);
    CK(cudaStreamSynchronize(c->cur));
    b = std::move(nb);
}

// prune_map's candidate draw (mapper.cpp:80-139), host side: candidates have topk_count <=
// threshold; ceil(keep_ratio * candidates) survive, drawn without replacement proportionally to
// max_contribution with std::mt19937_64(seed), uniformly once the mass is exhausted.
//
// The reference finds each weighted pick with a sequential scan of the remaining pool (fp64
// running sum, first position with u < acc) and erases it from a vector: O(C) per draw, O(C^2)
// per prune -- minutes to hours at config-3 candidate counts.  The same picks, bit for bit, in
// O(log C) per draw: Fenwick trees over the candidate order hold the pool membership and the
// pool scores.  A Fenwick descent locates the position p where the pool's prefix sum passes u;
// the pick is certain when u clears both of p's prefix bounds by B, a bound on |sequential fp64
// running sum - Fenwick prefix sum| (both are sums of <= C non-negative terms of total <= total:
// each within ~C eps total of the exact sum).  Only when u falls within B of a boundary, or past
// the pool's end (the reference's "no break: last pool element" case), does the draw replay the
// reference's scan exactly over the current pool.  Uniform draws pick the (rng() % size)-th pool
// element by a count descent.  Negative or non-finite scores take the reference loop verbatim.
struct Fenwick {
    std::vector<double> s;
    std::vector<int32_t> c;
    size_t n = 0, top = 1;
    explicit Fenwick(const std::vector<double>& v) : s(v.size() + 1, 0.0), c(v.size() + 1, 0), n(v.size()) {
        for (size_t i = 1; i <= n; ++i) {
            s[i] += v[i - 1];
            c[i] += 1;
            const size_t j = i + (i & (~i + 1));
            if (j <= n) {
                s[j] += s[i];
                c[j] += c[i];
            }
        }
        while (top * 2 <= n) top *= 2;
    }
    void rebuild_counts(const std::vector<uint8_t>& gone) {  // membership = !gone
        std::fill(c.begin(), c.end(), 0);
        for (size_t i = 1; i <= n; ++i) {
            c[i] += gone[i - 1] ? 0 : 1;
            const size_t j = i + (i & (~i + 1));
            if (j <= n) c[j] += c[i];
        }
    }
    void remove(size_t i, double v) {
        for (size_t k = i + 1; k <= n; k += k & (~k + 1)) {
            s[k] -= v;
            c[k] -= 1;
        }
    }
    double prefix(size_t i) const {  // sum over positions < i
        double r = 0.0;
        for (size_t k = i; k > 0; k -= k & (~k + 1)) r += s[k];
        return r;
    }
    size_t first_above(double u) const {  // first position whose inclusive prefix sum exceeds u (n: none)
        size_t pos = 0;
        double rem = u;
        for (size_t st = top; st > 0; st >>= 1)
            if (pos + st <= n && s[pos + st] <= rem) {
                pos += st;
                rem -= s[pos];
            }
        return pos;
    }
    size_t kth(size_t k) const {  // position of the k-th (0-based) pool member
        size_t pos = 0;
        int64_t rem = static_cast<int64_t>(k);
        for (size_t st = top; st > 0; st >>= 1)
            if (pos + st <= n && c[pos + st] <= rem) {
                pos += st;
                rem -= c[pos];
            }
        return pos;
    }
};

std::vector<int32_t> prune_select(const std::vector<int32_t>& counts, const std::vector<double>& maxc,
                                  double keep_ratio, uint64_t seed, int32_t threshold) {
    std::vector<int32_t> cand;
    for (size_t i = 0; i < counts.size(); ++i)
        if (counts[i] <= threshold) cand.push_back(static_cast<int32_t>(i));
    std::vector<int32_t> removed;
    if (cand.empty()) return removed;
    std::vector<double> score(cand.size());
    double total = 0.0;
    bool plain = true;  // every score finite and >= 0: the fast draw applies
    for (size_t i = 0; i < cand.size(); ++i) {
        score[i] = maxc[cand[i]];
        total += score[i];
        plain = plain && std::isfinite(score[i]) && score[i] >= 0.0;
    }
    if (!(total > 0.0)) return removed;  // survival weights undefined: keep every candidate
    const size_t keep = static_cast<size_t>(std::ceil(keep_ratio * static_cast<double>(cand.size())));
    if (keep >= cand.size()) return removed;
    const size_t C = cand.size();
    std::mt19937_64 rng(seed);
    std::vector<uint8_t> kept(C, 0);
    double mass = total;
    if (!plain || !std::isfinite(total)) {  // the reference loop verbatim
        std::vector<size_t> pool(C);
        for (size_t i = 0; i < C; ++i) pool[i] = i;
        for (size_t draw = 0; draw < keep; ++draw) {
            size_t pick = 0;
            if (mass > 0.0) {
                const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53 * mass;  // canonical_unit * mass
                double acc = 0.0;
                pick = pool.size() - 1;
                for (size_t q = 0; q < pool.size(); ++q) {
                    acc += score[pool[q]];
                    if (u < acc) {
                        pick = q;
                        break;
                    }
                }
            } else {
                pick = static_cast<size_t>(rng() % pool.size());
            }
            const size_t chosen = pool[pick];
            kept[chosen] = 1;
            mass -= score[chosen];
            if (mass < 0.0) mass = 0.0;
            pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(pick));
        }
    } else {
        // Error bound of both running sums against the exact pool sum: <= (2C + C + 128) eps S, S =
        // the pool sum when the tree was (re)built (subtractions leave errors of that size behind);
        // the tree is rebuilt from the remaining scores whenever the pool sum falls below S / 16, so
        // the bound stays within 16x of the current mass.
        // TK_PRUNE_BOUND_SCALE (tests only) widens the bound to force the exact fallback path
        const char* bs = std::getenv("TK_PRUNE_BOUND_SCALE");
        const double scale = bs ? std::max(1.0, std::atof(bs)) : 1.0;
        std::vector<double> live(score);
        std::vector<size_t> positive;  // the exact fallback scans only these: adding 0.0 is exact
        for (size_t i = 0; i < C; ++i)
            if (score[i] > 0.0) positive.push_back(i);
        Fenwick fw(live);
        double built_sum = fw.prefix(C);
        double bound = scale * 1.02 * (3.0 * static_cast<double>(C) + 128.0) * 0x1.0p-53 * built_sum;
        size_t pool_n = C;
        for (size_t draw = 0; draw < keep; ++draw) {
            size_t chosen = C;
            if (mass > 0.0) {
                const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53 * mass;
                const size_t p = fw.first_above(u);
                if (p < C && !kept[p] && score[p] > 0.0) {
                    const double lo = fw.prefix(p), hi = lo + score[p];
                    if (lo + bound <= u && u < hi - bound) chosen = p;
                }
                if (chosen == C) {  // within rounding reach of a boundary: the reference's scan
                    double acc = 0.0;
                    for (size_t q : positive) {
                        if (kept[q]) continue;
                        acc += score[q];
                        if (u < acc) {
                            chosen = q;
                            break;
                        }
                    }
                    if (chosen == C) chosen = fw.kth(pool_n - 1);  // no break: the pool's last element
                }
            } else {
                chosen = fw.kth(static_cast<size_t>(rng() % pool_n));
            }
            kept[chosen] = 1;
            fw.remove(chosen, score[chosen]);
            live[chosen] = 0.0;
            --pool_n;
            mass -= score[chosen];
            if (mass < 0.0) mass = 0.0;
            if (score[chosen] > 0.0 && fw.prefix(C) < built_sum * (1.0 / 16.0) && pool_n > 0) {
                fw = Fenwick(live);
                fw.rebuild_counts(kept);
                built_sum = fw.prefix(C);
                bound = scale * 1.02 * (3.0 * static_cast<double>(C) + 128.0) * 0x1.0p-53 * built_sum;
                std::vector<size_t> still;
                for (size_t q : positive)
                    if (!kept[q]) still.push_back(q);
                positive.swap(still);
            }
        }
    }
    for (size_t i = 0; i < C; ++i)
        if (!kept[i]) removed.push_back(cand[i]);
    return removed;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ mapping iteration
void tk_default_mapper_config(tk_mapper_config* cfg) {
    cfg->lambda_geo = 1.0;  // losses.hpp:9-21
    cfg->lambda_feat = 1.0;
    cfg->lambda1 = 0.2;
    cfg->lambda2 = 1.0;
    cfg->color_secondary = 0;
    cfg->feature_update_period = 5;  // mapper.hpp:16
    cfg->l1_deadband = 0.0;
    cfg->lr_mean = 2e-3;  // optimizer.hpp:15-22
    cfg->lr_log_scale = 5e-3;
    cfg->lr_rotation = 1e-3;
    cfg->lr_opacity = 5e-2;
    cfg->lr_color = 2e-2;
    cfg->lr_feature = 1e-2;
    cfg->beta1 = 0.9;  // optimizer.hpp:9-13
    cfg->beta2 = 0.999;
    cfg->eps = 1e-8;
    cfg->min_log_scale = -10.0;  // mapper.hpp:31-32
    cfg->max_log_scale = 1.0;
}

tk_status tk_keyframe_set(tk_ctx* c, int32_t slot, const tk_pose* pose, const tk_frame_view* fr) {
    return guarded([&] {
        if (!c || !pose || !fr) fail(TK_ERR_BAD_ARG, "null argument");
        if (slot < 0 || slot > (1 << 20)) fail(TK_ERR_BAD_ARG, "keyframe slot out of range");
        if (fr->width <= 0 || fr->height <= 0 || fr->d < 0) fail(TK_ERR_BAD_ARG, "bad frame shape");
        if (!fr->color || !fr->depth) fail(TK_ERR_BAD_ARG, "frame needs color and depth");
        if (fr->d > 0 && !fr->feature) fail(TK_ERR_BAD_ARG, "frame feature is NULL but d > 0");
        CK(cudaSetDevice(c->device));
        on_main(c);
        if (static_cast<size_t>(slot) >= c->kfs.size()) c->kfs.resize(slot + 1);
        Keyframe& k = c->kfs[slot];
        k.pose = *pose;
        k.w = fr->width;
        k.h = fr->height;
        k.d = fr->d;
        k.has_feature = fr->d > 0;
        const int64_t P = static_cast<int64_t>(k.w) * k.h;
        float* col = ensure<float>(k.color, P * 3);
        float* dep = ensure<float>(k.depth, P);
        copy_in(col, fr->color, P * 3 * sizeof(float), fr->mem, c);
        copy_in(dep, fr->depth, P * sizeof(float), fr->mem, c);
        float* feat = nullptr;
        if (k.has_feature) {
            feat = ensure<float>(k.feature, P * k.d);
            copy_in(feat, fr->feature, static_cast<size_t>(P) * k.d * sizeof(float), fr->mem, c);
        }
        uint8_t* valid = ensure<uint8_t>(k.valid, P);
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        tk::launch_gt_valid(feat, P, k.d, valid, dscal + 9, dep, c->cur);
        CK_LAUNCH(c);
        if (c->comm)  // D-sharded: a pixel's keyframe row is valid if any shard's channels are non-zero
            NK(g_nccl.AllReduce(valid, valid, static_cast<size_t>(P), ncclUint8, ncclMax, c->comm, c->cur));
        tk::copy_words_to_mapped(c->hscal_dev + 9, dscal + 9, 1, c->cur);
        sync(c);
        k.depth_n = c->hscal[9];
        main_done(c);
    });
}

tk_status tk_optimizer_reset(tk_ctx* c, int32_t reset_stats) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);  // pending lazy steps land before the moments are dropped
        const int64_t n = c->n;
        const int dims[5] = {3, 3, 4, 1, 3};
        for (int g = 0; g < 5; ++g) {
            CK(cudaMemsetAsync(ensure<double>(c->am[g], n * dims[g]), 0, std::max<int64_t>(n, 1) * dims[g] * 8, c->cur));
            CK(cudaMemsetAsync(ensure<double>(c->av[g], n * dims[g]), 0, std::max<int64_t>(n, 1) * dims[g] * 8, c->cur));
        }
        const int64_t nd = n * std::max(c->d, 1);
        CK(cudaMemsetAsync(ensure<float>(c->fm, nd), 0, std::max<int64_t>(nd, 1) * 4, c->cur));
        CK(cudaMemsetAsync(ensure<float>(c->fv, nd), 0, std::max<int64_t>(nd, 1) * 4, c->cur));
        if (reset_stats || c->stat_n != n) {
            CK(cudaMemsetAsync(ensure<int32_t>(c->stat_count, n), 0, std::max<int64_t>(n, 1) * 4, c->cur));
            CK(cudaMemsetAsync(ensure<double>(c->stat_maxc, n), 0, std::max<int64_t>(n, 1) * 8, c->cur));
            c->stat_n = n;
        }
        c->step_geo = c->step_feat = 0;
        tk::launch_fill_i32(ensure<int32_t>(c->f_last, n), n, 0, c->cur);
        c->f_tab_host.assign(1, tk::AdamStepParams{});  // index 0 unused: steps are 1-based
        c->feat_stale = false;
        c->opt_ready = true;
        c->opt_n = n;
        c->opt_d = c->d;
        main_done(c);
    });
}

tk_status tk_optimize_step(tk_ctx* c, const tk_mapper_config* cfg, const tk_camera* cam, const tk_settings* s,
                           int32_t slot, int64_t iteration, double* values_out, int32_t* feature_step_out) {
    return guarded([&] {
        check_frame(cam, s);
        if (!cfg) fail(TK_ERR_BAD_ARG, "null mapper config");
        if (c->band_n > 1) fail(TK_ERR_STATE, "optimize_step: the geometry split (tk_geometry_band) is frame-API only");
        if (slot < 0 || static_cast<size_t>(slot) >= c->kfs.size() || c->kfs[slot].w == 0)
            fail(TK_ERR_BAD_ARG, "optimize_step: no keyframe in that slot");
        if (cfg->feature_update_period <= 0) fail(TK_ERR_BAD_ARG, "feature_update_period must be positive");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if (!c->opt_ready || c->opt_n != c->n || c->opt_d != c->d || c->stat_n != c->n)
            fail(TK_ERR_STATE, "optimizer state does not match the scene (tk_optimizer_reset)");
        const Keyframe& kf = c->kfs[slot];
        if (kf.w != cam->width || kf.h != cam->height)
            fail(TK_ERR_BAD_ARG, "compute_losses: render/frame shape mismatch");
        const bool feature_step = (iteration % cfg->feature_update_period) == 0;  // mapper.cpp:171
        const bool sharded = c->comm != nullptr;  // D-sharded mapping (features: this rank's slice)
        const bool use_ssim = cfg->lambda1 != 0.0 && cfg->color_secondary == 0;
        if (use_ssim && (cam->width < tk::kSsimWin || cam->height < tk::kSsimWin))
            fail(TK_ERR_BAD_ARG, "ssim: image smaller than the 11x11 window");
        if (feature_step) {
            if (c->d <= 0 || !c->has_features)
                fail(TK_ERR_BAD_ARG, "compute_losses: feature loss requested but render has no feature image");
            if (kf.d != c->d) fail(TK_ERR_BAD_ARG, "compute_losses: feature shape mismatch");
        }
        // Lazy feature Adam (TK_LAZY_ADAM=0: eager): a feature step updates only the rows this
        // frame's records reach; the other rows' zero-gradient steps are replayed bit-identically
        // (k_feature_catchup) right before anything reads them.
        static const bool lazy_env = [] {
            const char* e = std::getenv("TK_LAZY_ADAM");
            return !(e && e[0] == '0');
        }();
        const bool lazy_feat = feature_step && lazy_env && !sharded && c->d % 4 == 0 && c->d <= 512;
        CK(cudaSetDevice(c->device));
        on_main(c);
        cudaStream_t st = c->cur;
        // render_geometric on the keyframe pose (mapper.cpp:173)
        prepare(c, &kf.pose, cam, s);
        forward(c, cam, s, true);
        const tk::Frame f = make_frame(c, cam, s);
        const int64_t P = static_cast<int64_t>(f.width) * f.height;
        const int64_t n = c->n;
        const int d = c->d;
        double* gc = ensure<double>(c->l_gc, P * 3);
        double* gd = ensure<double>(c->l_gd, P);
        double* partial = ensure<double>(c->l_partial, tk::kLossBlocks * tk::kLossSlots);
        double* values = ensure<double>(c->l_values, 4);
        float* fscale = ensure<float>(c->l_fscale, 1);
        const int wpp = (d + 15) / 16;
        uint32_t* signs = feature_step ? ensure<uint32_t>(c->l_signs, P * std::max(wpp, 1)) : nullptr;
        // this feature step's Adam constants (step k, 1-based), kept per step for lazy replays
        const int64_t kstep = c->step_feat + 1;
        tk::AdamStepParams ast{};
        if (feature_step && d > 0) {
            ast.lr = static_cast<float>(cfg->lr_feature);
            ast.beta1 = static_cast<float>(cfg->beta1);
            ast.beta2 = static_cast<float>(cfg->beta2);
            ast.eps = static_cast<float>(cfg->eps);
            ast.one_m_beta1 = static_cast<float>(1.0 - cfg->beta1);
            ast.one_m_beta2 = static_cast<float>(1.0 - cfg->beta2);
            ast.inv_bc1 = static_cast<float>(1.0 / (1.0 - std::pow(cfg->beta1, static_cast<double>(kstep))));
            ast.inv_bc2 = static_cast<float>(1.0 / (1.0 - std::pow(cfg->beta2, static_cast<double>(kstep))));
            // a step that failed after recording its constants left an extra entry: drop it
            if (c->f_tab_host.size() < static_cast<size_t>(kstep)) fail(TK_ERR_STATE, "feature step table out of sync");
            c->f_tab_host.resize(static_cast<size_t>(kstep));
            c->f_tab_host.push_back(ast);
            const int64_t cap = static_cast<int64_t>(c->f_tab.bytes / sizeof(tk::AdamStepParams));
            tk::AdamStepParams* tab = cap > kstep ? ptr<tk::AdamStepParams>(c->f_tab)
                                                  : grow_keep<tk::AdamStepParams>(c, c->f_tab, kstep, 2 * kstep + 64, false);
            CK(cudaMemcpyAsync(tab + kstep, &c->f_tab_host[kstep], sizeof(tk::AdamStepParams), cudaMemcpyHostToDevice,
                               st));
        }
        // lazy: the rows this frame's records reach catch up to step k-1 before the loss reads them
        SlotIndex early_si{};
        bool have_si = false;
        if (lazy_feat) {
            Records r;
            r.w = f.width;
            r.h = f.height;
            r.k = f.k;
            r.index = ptr<int32_t>(c->o_index);
            r.weight = ptr<double>(c->o_weight);
            r.count = ptr<uint8_t>(c->o_count);
            early_si = build_slot_index(c, r);
            have_si = true;
            tk::launch_active_rows(early_si.seg, n, ensure<int32_t>(c->f_active, n), ensure<int32_t>(c->f_active_n, 1),
                                   st);
            tk::FeatAdamParams fa{};
            fa.active = ptr<int32_t>(c->f_active);
            fa.n_active = ptr<int32_t>(c->f_active_n);
            fa.n = n;
            fa.d = d;
            fa.seg = early_si.seg;
            fa.feat = ptr<float>(c->feature);
            fa.m = ptr<float>(c->fm);
            fa.v = ptr<float>(c->fv);
            fa.last = ptr<int32_t>(c->f_last);
            fa.tab = ptr<tk::AdamStepParams>(c->f_tab);
            if (c->feat_stale) {
                tk::launch_feature_catchup(fa, static_cast<int>(kstep - 1), true, st);
            }
        } else if (feature_step && d > 0) {
            flush_features(c);  // an eager step needs every row at step k-1 (step_feat is still k-1)
        }
        {
            PhaseScope phase(c, TK_PHASE_LOSS);
            CK(cudaMemsetAsync(partial, 0, tk::kLossBlocks * tk::kLossSlots * sizeof(double), st));
            tk::launch_topk_stats(ptr<int32_t>(c->o_index), ptr<uint8_t>(c->o_count), P, f.k,
                                  ptr<int32_t>(c->stat_count), st);
            // compute_losses (mapper.cpp:176, losses.cpp:22-133)
            tk::ColorLossParams lp{};
            lp.w = f.width;
            lp.h = f.height;
            lp.color = ptr<double>(c->o_color);
            lp.depth = ptr<double>(c->o_depth);
            lp.gt_color = ptr<float>(kf.color);
            lp.gt_depth = ptr<float>(kf.depth);
            lp.lambda_geo = cfg->lambda_geo;
            lp.lambda1 = cfg->lambda1;
            lp.lambda2 = cfg->lambda2;
            lp.deadband = cfg->l1_deadband;
            lp.use_ssim = use_ssim ? 1 : 0;
            lp.use_depth = (kf.depth_n > 0 && cfg->lambda2 != 0.0) ? 1 : 0;
            lp.inv_color_n = 1.0 / (static_cast<double>(f.width) * f.height * 3.0);
            lp.inv_depth_n = kf.depth_n > 0 ? 1.0 / static_cast<double>(kf.depth_n) : 0.0;
            {
                const int ow = f.width - tk::kSsimWin + 1, oh = f.height - tk::kSsimWin + 1;
                const size_t count = use_ssim ? static_cast<size_t>(ow) * oh * 3 : 1;  // ssim.cpp:119-123
                lp.inv_count = 1.0 / static_cast<double>(count);
                double sum = 0.0;  // gaussian_kernel(), ssim.cpp:18-28
                for (int i = 0; i < tk::kSsimWin; ++i) {
                    const double dd = i - tk::kSsimWin / 2;
                    lp.kern[i] = std::exp(-0.5 * dd * dd / (1.5 * 1.5));
                    sum += lp.kern[i];
                }
                for (double& v : lp.kern) v /= sum;
                if (use_ssim) {
                    lp.win = ensure<double>(c->ssim_win, 15LL * oh * ow);
                }
            }
            lp.grad_color = gc;
            lp.grad_depth = gd;
            lp.partial = partial;
            tk::launch_color_loss(lp, st);
            if (feature_step) {
                tk::FeatLossParams fl{};
                fl.width = f.width;
                fl.height = f.height;
                fl.k = f.k;
                fl.d = d;
                fl.index = ptr<int32_t>(c->o_index);
                fl.weight = ptr<double>(c->o_weight);
                fl.count = ptr<uint8_t>(c->o_count);
                fl.feat = ptr<float>(c->feature);
                fl.gt = ptr<float>(kf.feature);
                fl.gt_valid = ptr<uint8_t>(kf.valid);
                fl.signs = signs;
                fl.partial = partial;
                tk::launch_feature_loss(fl, st);
            }
            if (sharded)  // feature partials differ per shard; colour / depth rows are replicas
                NK(g_nccl.AllReduce(partial, partial, tk::kLossBlocks * tk::kLossSlots, ncclFloat64, ncclSum, c->comm,
                                    st));
            tk::FinalizeParams fp{};
            fp.partial = partial;
            fp.nparts = tk::kLossBlocks;
            fp.replicas = sharded ? static_cast<double>(c->nranks) : 1.0;
            fp.lambda_geo = cfg->lambda_geo;
            fp.lambda_feat = cfg->lambda_feat;
            fp.lambda1 = cfg->lambda1;
            fp.lambda2 = cfg->lambda2;
            fp.use_ssim = lp.use_ssim;
            fp.secondary_l1 = (cfg->lambda1 != 0.0 && cfg->color_secondary != 0) ? 1 : 0;
            fp.use_depth = lp.use_depth;
            fp.feature_step = feature_step ? 1 : 0;
            fp.d = sharded ? c->d_total : d;  // losses.cpp:106: mean over every channel
            fp.inv_color_n = lp.inv_color_n;
            fp.inv_depth_n = lp.inv_depth_n;
            fp.inv_count = lp.inv_count;
            fp.values = values;
            fp.feat_scale = fscale;
            tk::launch_loss_finalize(fp, st);
            CK_LAUNCH(c);
        }
        tk::copy_words_to_mapped(c->hvals_dev, values, 3, st);
        c->has_values = true;
        // the feature half first (mapper.cpp:239-252; independent of the geometry half): its
        // sign image was just written by the loss and is still in L2 for the record sweep
        {
            PhaseScope phase(c, TK_PHASE_ADAM);
            if (feature_step && d > 0) {  // mapper.cpp:239-252
                c->step_feat = kstep;
                Records r;
                r.w = f.width;
                r.h = f.height;
                r.k = f.k;
                r.index = ptr<int32_t>(c->o_index);
                r.weight = ptr<double>(c->o_weight);
                r.count = ptr<uint8_t>(c->o_count);
                const SlotIndex si = have_si ? early_si : build_slot_index(c, r);
                tk::FeatAdamParams fa{};
                fa.n = n;
                fa.k = f.k;
                fa.d = d;
                fa.seg = si.seg;
                fa.slots = si.slots;
                fa.wnorm = si.wnorm;
                fa.signs = signs;
                fa.scale = fscale;
                fa.feat = ptr<float>(c->feature);
                fa.m = ptr<float>(c->fm);
                fa.v = ptr<float>(c->fv);
                fa.st = ast;
                fa.plan = si.plan;
                if (sharded) fa.row_ss = ensure<float>(c->row_ss, n);
                fa.last = ptr<int32_t>(c->f_last);
                fa.cur = static_cast<int>(kstep);
                fa.tab = ptr<tk::AdamStepParams>(c->f_tab);
                fa.lazy = lazy_feat ? 1 : 0;
                if (lazy_feat) {
                    fa.active = ptr<int32_t>(c->f_active);
                    fa.n_active = ptr<int32_t>(c->f_active_n);
                    // active rows <= rows with records <= min(n, record slots)
                    const int64_t cap = std::min<int64_t>(n, static_cast<int64_t>(P) * f.k);
                    fa.grad = ensure<float>(c->f_active_grad, std::max<int64_t>(cap, 1) * d);
                    fa.cap_active = cap;
                }
                if (lazy_feat && !tk::feature_adam_lazy_ok(fa)) fail(TK_ERR_STATE, "lazy feature Adam: bad layout");
                tk::launch_feature_adam(fa, st);
                if (fa.lazy) c->feat_stale = true;
                if (sharded) {  // mapper.cpp:249: the norm of the whole row, over every shard
                    NK(g_nccl.AllReduce(fa.row_ss, fa.row_ss, static_cast<size_t>(n), ncclFloat32, ncclSum, c->comm,
                                        st));
                    tk::launch_feature_renorm(ptr<float>(c->feature), fa.row_ss, n, d, st);
                }
                CK_LAUNCH(c);
            }
        }
        // backward_geometric (mapper.cpp:179-180) on this forward
        double* mid = geom_sweep(c, f, gc, gd);
        // The fixed-order merge makes every replica's geometry gradient bit-identical, so the
        // D-sharded step needs no collective here; the atomic flush (TK_GEOM_BWD_ATOMIC=1) is
        // order-dependent and all-reduces it so the replicas cannot drift.
        const bool geo_allreduce = sharded && c->geom_atomic;
        if (geo_allreduce)
            NK(g_nccl.AllReduce(mid, mid, static_cast<size_t>(n) * 10, ncclFloat64, ncclSum, c->comm, st));
        {
            PhaseScope phase(c, TK_PHASE_ADAM);
            // geometry groups (mapper.cpp:183-236): five adam_step calls, one step counter each
            c->step_geo += 1;
            tk::GeoAdamParams ga{};
            ga.mean = ptr<double>(c->mean);
            ga.log_scale = ptr<double>(c->log_scale);
            ga.rotation = ptr<double>(c->rotation);
            ga.opacity_logit = ptr<double>(c->opacity_logit);
            ga.color = ptr<double>(c->color);
            for (int g = 0; g < 5; ++g) {
                ga.m[g] = ptr<double>(c->am[g]);
                ga.v[g] = ptr<double>(c->av[g]);
            }
            ga.lr[0] = cfg->lr_mean;
            ga.lr[1] = cfg->lr_log_scale;
            ga.lr[2] = cfg->lr_rotation;
            ga.lr[3] = cfg->lr_opacity;
            ga.lr[4] = cfg->lr_color;
            ga.beta1 = cfg->beta1;
            ga.beta2 = cfg->beta2;
            ga.eps = cfg->eps;
            ga.bc1 = 1.0 - std::pow(cfg->beta1, static_cast<double>(c->step_geo));  // optimizer.cpp:52-53
            ga.bc2 = 1.0 - std::pow(cfg->beta2, static_cast<double>(c->step_geo));
            ga.min_log_scale = cfg->min_log_scale;
            ga.max_log_scale = cfg->max_log_scale;
            ga.contrib = ptr<unsigned long long>(c->o_contrib);
            ga.max_contrib = ptr<double>(c->stat_maxc);
            tk::ChainParams cp = chain_params(c, &kf.pose, cam, s, mid);
            cp.mid_scale = geo_allreduce ? 1.0 / c->nranks : 1.0;
            cp.g_mean = ensure<double>(c->gg_mean, n * 3);
            cp.g_log_scale = ensure<double>(c->gg_ls, n * 3);
            cp.g_rotation = ensure<double>(c->gg_rot, n * 4);
            cp.g_opacity_logit = ensure<double>(c->gg_op, n);
            cp.g_color = ensure<double>(c->gg_col, n * 3);
            cp.twist = nullptr;
            tk::launch_chain(cp, st);
            ga.g[0] = cp.g_mean;
            ga.g[1] = cp.g_log_scale;
            ga.g[2] = cp.g_rotation;
            ga.g[3] = cp.g_opacity_logit;
            ga.g[4] = cp.g_color;
            tk::launch_geo_adam(ga, n, st);
            CK_LAUNCH(c);

        }
        // the scene changed: the next render re-projects (records keep the pre-step snapshot)
        c->scene_version += 1;
        c->prepared = false;
        c->aux_valid = false;
        if (feature_step_out) *feature_step_out = feature_step ? 1 : 0;
        if (values_out) {
            sync(c);
            std::memcpy(values_out, c->hvals, 3 * sizeof(double));
        }
        main_done(c);
    });
}

tk_status tk_optimizer_flush(tk_ctx* c) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);
        main_done(c);
    });
}

tk_status tk_loss_values(tk_ctx* c, double values[3]) {
    return guarded([&] {
        if (!c->has_values) fail(TK_ERR_STATE, "no optimize_step has run");
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        std::memcpy(values, c->hvals, 3 * sizeof(double));
    });
}

tk_status tk_scene_download(tk_ctx* c, const tk_scene_out* o) {
    return guarded([&] {
        if (!c || !o) fail(TK_ERR_BAD_ARG, "null argument");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if ((o->topk_count || o->max_contribution) && c->stat_n != c->n)
            fail(TK_ERR_STATE, "no selection statistics for this scene (tk_optimizer_reset)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);  // lazily optimised feature rows must be current
        const int64_t n = c->n;
        copy_out(o->mean, c->mean.p, n * 3 * sizeof(double), o->mem, c);
        copy_out(o->log_scale, c->log_scale.p, n * 3 * sizeof(double), o->mem, c);
        copy_out(o->rotation, c->rotation.p, n * 4 * sizeof(double), o->mem, c);
        copy_out(o->opacity_logit, c->opacity_logit.p, n * sizeof(double), o->mem, c);
        copy_out(o->color, c->color.p, n * 3 * sizeof(double), o->mem, c);
        if (o->feature && c->has_features)
            copy_out(o->feature, c->feature.p, static_cast<size_t>(n) * c->d * sizeof(float), o->mem, c);
        copy_out(o->topk_count, c->stat_count.p, n * sizeof(int32_t), o->mem, c);
        copy_out(o->max_contribution, c->stat_maxc.p, n * sizeof(double), o->mem, c);
        if (o->mem == TK_HOST) sync(c);
        main_done(c);
    });
}

// ------------------------------------------------------------------ structural edits
tk_status tk_scene_info(tk_ctx* c, int64_t* n, int32_t* d, uint64_t* generation) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (n) *n = c->n;
        if (d) *d = c->d;
        if (generation) *generation = c->generation;
    });
}

tk_status tk_insert_gaussians(tk_ctx* c, const tk_source_view* src, double tau, const tk_pose* w2c,
                              int32_t* inserted) {
    return guarded([&] {
        if (!c || !src || !w2c) fail(TK_ERR_BAD_ARG, "null argument");
        if (src->n < 0 || src->d < 0) fail(TK_ERR_BAD_ARG, "negative source size");
        if (src->n > 0 && (!src->position || !src->color || !src->spacing || !src->distance))
            fail(TK_ERR_BAD_ARG, "insert_gaussians: position, color, spacing and distance are required");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);  // lazily optimised feature rows must be current
        cudaStream_t st = c->cur;
        const int64_t ns = src->n;
        if (inserted) *inserted = 0;
        if (ns == 0) {
            main_done(c);
            return;
        }
        DevBuf bpos, bcol, bsp, bdist, bfeat, bflag, bflag32, bslot;
        auto dev_in = [&](DevBuf& b, const void* p, size_t bytes) -> const void* {
            if (src->mem == TK_DEVICE) return p;
            ensure<char>(b, bytes);
            copy_in(b.p, p, bytes, TK_HOST, c);
            return b.p;
        };
        const double* pos = static_cast<const double*>(dev_in(bpos, src->position, ns * 3 * sizeof(double)));
        const double* col = static_cast<const double*>(dev_in(bcol, src->color, ns * 3 * sizeof(double)));
        const double* sp = static_cast<const double*>(dev_in(bsp, src->spacing, ns * sizeof(double)));
        const double* dist = static_cast<const double*>(dev_in(bdist, src->distance, ns * sizeof(double)));
        const float* feat = (src->feature && src->d > 0)
                                ? static_cast<const float*>(dev_in(bfeat, src->feature, ns * src->d * sizeof(float)))
                                : nullptr;
        uint8_t* flag = ensure<uint8_t>(bflag, ns);
        int32_t* flag32 = ensure<int32_t>(bflag32, ns);
        int32_t* slot = ensure<int32_t>(bslot, ns);
        tk::launch_insert_flags(dist, ns, tau, flag, flag32, st);
        ensure_scratch(c, ns + 1);
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        tk::scan_exclusive(flag32, slot, ns, dscal + 10, c->scratch.p, st);
        tk::copy_words_to_mapped(c->hscal_dev + 10, dscal + 10, 1, st);
        sync(c);
        const int64_t total = c->hscal[10];
        if (total > 0) {
            if (c->d == 0 && feat && (c->n == 0 || !c->has_features)) c->d = src->d;  // mapper.cpp:40-41
            const int64_t n0 = c->n, n1 = n0 + total;
            const int d = c->d;
            tk::InsertParams ip{};
            ip.n_src = ns;
            ip.base = n0;
            ip.position = pos;
            ip.color = col;
            ip.feature = feat;
            ip.d_src = src->d;
            ip.spacing = sp;
            ip.slot = slot;
            ip.flag = flag;
            // se3_inverse (pose.cpp:14-19) and its normalised rotation (mapper.cpp:25-26)
            const double qi[4] = {w2c->qw, -w2c->qx, -w2c->qy, -w2c->qz};
            const double t[3] = {w2c->tx, w2c->ty, w2c->tz};
            double ti[3];
            tk::quat_rotate_eigen(qi, t, ti);
            const double qn = std::sqrt(((qi[0] * qi[0] + qi[1] * qi[1]) + qi[2] * qi[2]) + qi[3] * qi[3]);
            for (int a = 0; a < 4; ++a) {
                ip.qi[a] = qi[a];
                ip.rot[a] = qi[a] / qn;
            }
            for (int a = 0; a < 3; ++a) ip.ti[a] = -ti[a];
            ip.opacity_logit = std::log(0.5 / (1.0 - 0.5));                     // logit(0.5)
            ip.d = d;
            ip.mean = grow_keep<double>(c, c->mean, n0 * 3, n1 * 3, false);
            ip.log_scale = grow_keep<double>(c, c->log_scale, n0 * 3, n1 * 3, false);
            ip.rotation = grow_keep<double>(c, c->rotation, n0 * 4, n1 * 4, false);
            ip.opacity = grow_keep<double>(c, c->opacity_logit, n0, n1, false);
            ip.color_out = grow_keep<double>(c, c->color, n0 * 3, n1 * 3, false);
            if (d > 0) {
                ip.feat = grow_keep<float>(c, c->feature, c->has_features ? n0 * d : 0, n1 * d, false);
                c->has_features = true;
            }
            tk::launch_insert_fill(ip, st);
            CK_LAUNCH(c);
            if (c->opt_ready && c->opt_n == n0) {  // OptimizerState::extend (optimizer.cpp:29-36)
                const int dims[5] = {3, 3, 4, 1, 3};
                for (int g = 0; g < 5; ++g) {
                    grow_keep<double>(c, c->am[g], n0 * dims[g], n1 * dims[g], true);
                    grow_keep<double>(c, c->av[g], n0 * dims[g], n1 * dims[g], true);
                }
                grow_keep<float>(c, c->fm, n0 * c->opt_d, n1 * d, true);
                grow_keep<float>(c, c->fv, n0 * c->opt_d, n1 * d, true);
                if (c->opt_d != d) {  // the feature group is sized now (mapper.cpp:54)
                    CK(cudaMemsetAsync(c->fm.p, 0, n1 * d * sizeof(float), st));
                    CK(cudaMemsetAsync(c->fv.p, 0, n1 * d * sizeof(float), st));
                }
                c->opt_n = n1;
                c->opt_d = d;
                // every row is current (flushed on entry); the new rows start at this step
                tk::launch_fill_i32(ensure<int32_t>(c->f_last, n1), n1, static_cast<int32_t>(c->step_feat), st);
            }
            if (c->stat_n == n0) {
                grow_keep<int32_t>(c, c->stat_count, n0, n1, true);
                grow_keep<double>(c, c->stat_maxc, n0, n1, true);
                c->stat_n = n1;
            }
            c->n = n1;
            c->generation += 1;                                                 // mapper.cpp:56
            scene_changed(c);
            if (inserted) *inserted = static_cast<int32_t>(total);
        }
        sync(c);
        for (DevBuf* b : {&bpos, &bcol, &bsp, &bdist, &bfeat, &bflag, &bflag32, &bslot}) b->release();
        main_done(c);
    });
}

tk_status tk_prune_draw(const int32_t* topk_count, const double* max_contribution, int64_t n, double keep_ratio,
                        uint64_t seed, int32_t threshold, int32_t* removed_out, int64_t* n_removed) {
    return guarded([&] {
        if (n < 0 || (n > 0 && (!topk_count || !max_contribution))) fail(TK_ERR_BAD_ARG, "bad statistics arrays");
        std::vector<int32_t> counts(topk_count, topk_count + n);
        std::vector<double> maxc(max_contribution, max_contribution + n);
        const std::vector<int32_t> removed = prune_select(counts, maxc, keep_ratio, seed, threshold);
        if (removed_out && !removed.empty()) std::memcpy(removed_out, removed.data(), removed.size() * sizeof(int32_t));
        if (n_removed) *n_removed = static_cast<int64_t>(removed.size());
    });
}

tk_status tk_prune_map(tk_ctx* c, double keep_ratio, uint64_t seed, int32_t threshold, int32_t* removed_out,
                       int64_t* n_removed) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if (c->stat_n != c->n) fail(TK_ERR_STATE, "no selection statistics for this scene (tk_optimizer_reset)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);  // lazily optimised feature rows must be current
        cudaStream_t st = c->cur;
        const int64_t n = c->n;
        std::vector<int32_t> counts(n);
        std::vector<double> maxc(n);
        copy_out(counts.data(), c->stat_count.p, n * sizeof(int32_t), TK_HOST, c);
        copy_out(maxc.data(), c->stat_maxc.p, n * sizeof(double), TK_HOST, c);
        sync(c);
        const std::vector<int32_t> removed = prune_select(counts, maxc, keep_ratio, seed, threshold);
        const int64_t nr = static_cast<int64_t>(removed.size());
        if (nr > 0) {  // mapper.cpp:141-154 + OptimizerState::compact
            DevBuf brem, bkeep, bpos;
            int32_t* drem = ensure<int32_t>(brem, nr);
            copy_in(drem, removed.data(), nr * sizeof(int32_t), TK_HOST, c);
            int32_t* keep = ensure<int32_t>(bkeep, n);
            int32_t* pos = ensure<int32_t>(bpos, n);
            tk::launch_keep_flags(drem, nr, n, keep, st);
            ensure_scratch(c, n + 1);
            int64_t* dscal = ensure<int64_t>(c->dscal, 16);
            tk::scan_exclusive(keep, pos, n, dscal + 11, c->scratch.p, st);
            const int64_t nk = n - nr;
            compact_rows<double>(c, c->mean, n, 3, nk, keep, pos);
            compact_rows<double>(c, c->log_scale, n, 3, nk, keep, pos);
            compact_rows<double>(c, c->rotation, n, 4, nk, keep, pos);
            compact_rows<double>(c, c->opacity_logit, n, 1, nk, keep, pos);
            compact_rows<double>(c, c->color, n, 3, nk, keep, pos);
            if (c->has_features && c->d > 0) compact_rows<float>(c, c->feature, n, c->d, nk, keep, pos);
            if (c->opt_ready && c->opt_n == n) {
                const int dims[5] = {3, 3, 4, 1, 3};
                for (int g = 0; g < 5; ++g) {
                    compact_rows<double>(c, c->am[g], n, dims[g], nk, keep, pos);
                    compact_rows<double>(c, c->av[g], n, dims[g], nk, keep, pos);
                }
                if (c->opt_d > 0) {
                    compact_rows<float>(c, c->fm, n, c->opt_d, nk, keep, pos);
                    compact_rows<float>(c, c->fv, n, c->opt_d, nk, keep, pos);
                }
                c->opt_n = nk;
                // every row is current (flushed on entry)
                tk::launch_fill_i32(ensure<int32_t>(c->f_last, nk), nk, static_cast<int32_t>(c->step_feat), st);
            }
            sync(c);
            for (DevBuf* b : {&brem, &bkeep, &bpos}) b->release();
            c->n = nk;
            c->generation += 1;                                                 // mapper.cpp:153
            scene_changed(c);
        }
        // the statistics window restarts at every prune (mapper.cpp:156-159)
        CK(cudaMemsetAsync(c->stat_count.p, 0, std::max<int64_t>(c->n, 1) * sizeof(int32_t), st));
        CK(cudaMemsetAsync(c->stat_maxc.p, 0, std::max<int64_t>(c->n, 1) * sizeof(double), st));
        c->stat_n = c->n;
        if (removed_out && nr) std::memcpy(removed_out, removed.data(), nr * sizeof(int32_t));
        if (n_removed) *n_removed = nr;
        main_done(c);
    });
}

}  // extern "C"
