// hh_wy_flow.cuh -- K5f: the whole compact-WY block program as ONE dataflow launch.
// (Included by hh_wy.cu inside its anonymous namespace: it uses that file's constants,
// barrier structs and device helpers.)
//
// Why.  As separate launches, the projection G = W^T X (K5a) and the update X <- X - V G
// (K5b) move X three times per block: K5a reads it, K5b reads it again and writes it.  The
// method's cost model is one read and one write per vector ("4nh operations",
// P:284 "(8h+1)n"), so a one-block program moves 1.5x and a four-block one 6x the
// algorithmic bytes.  Here both roles run at the same time on disjoint CTAs of one launch
// and hand each 128-column tile from one to the other while the tile is still in L2:
//
//   * project CTAs (blockIdx < P) take (pass, tile, K chunk) units, each K chunk a slice
//     of the rows; the fp32 partial G of a unit goes to a slot, the last of a tile's
//     nkc units to arrive (atomic count) adds the slots in fixed order (deterministic),
//     writes G as bf16 hi/lo into a ring slot and raises the tile's `gready` flag;
//   * update CTAs take (pass, tile, row segment) units, wait for `gready`, load G and the
//     X rows (an L2 hit: the projection read them moments ago) and store Y; every stored
//     row chunk counts into the tile's `udone`;
//   * the next pass of a tile (multi-block programs) waits for `udone` of the previous pass,
//     so X stays L2-resident across all passes of a tile; a window of D tiles (a project
//     unit of tile t waits until tile t - D has left the program) bounds the L2 footprint.
//
// Units are dispensed in one global order -- pairs (pass q, tile t) by s = q + t, then t --
// round-robin over each role's CTAs; every wait is on a unit earlier in that order, so the
// program cannot deadlock as long as all CTAs are resident (cooperative launch, grid <= SMs).
// Correctness does not depend on L2 hits: a miss re-reads HBM.

constexpr int kFlowMaxPasses = kMaxPasses;

struct FlowPass {
    int wrow, wrow_lo, kw, wmap;   // project operand: W rows [wrow, +kw) (hi), lo rows; map 0/1
    int vmap, vrow_hi, vrow_lo;    // update operand: map 0 (V), 1 (Asym), 2 (V2), rows
    int ks0, rc0, xrc0;            // QR skips: first K step, first MMA row chunk, first row chunk
    int target;                    // udone count that completes a tile: (nrc - xrc0) * 4
    const float *dscale, *pre, *post;
};

struct FlowArgs {
    CUtensorMap mXp, mYp;   // project operand boxes (32 rows x 128 columns) of X / Y
    CUtensorMap mXu, mYu;   // update boxes of X / Y (SS: 128 x 16; TS: 32 x 128, SW128)
    CUtensorMap mW[2];      // W hi/lo, boxes 32 x b and 32 x 2b
    CUtensorMap mG;         // G ring, box 32 x 128 (SS update)
    CUtensorMap mV[3];      // V, Asym, V2 (boxes 32 x 128)
    uint16_t *ring;         // G ring: hi rows [0, D*128), lo rows [D*128, 2*D*128), pitch kwmax
    float *part;            // partials [D][nkc][kwmax/32][128][32]
    int *gcount, *gready, *udone;   // [np][ntiles]
    int64_t N;
    int n, n_pad, np, ntiles, D, P, nkc, rseg, kwmax, ts, nraw, nxs, sms, G;
    int pol;                     // L2 policy bits (A/B): 1 project evict_last, 2 update evict_first
    unsigned long long *tl;      // debug: per-CTA role timeline (hh_debug_wy_timeline), or NULL
    FlowPass pass[kFlowMaxPasses];
};

// debug timeline: per CTA 16 counters (cycles unless noted), written once at the end
enum : int {
    TL_ROLE = 0, TL_TOTAL, TL_PDEP, TL_PRING, TL_MMA_IN, TL_MMA_ACC, TL_EPI_ACC, TL_EPI_RED,
    TL_EPI_X, TL_UNITS, TL_CV_IN, TL_CV_OUT, TL_EPI_BUSY, TL_UDEP, TL_13, TL_14
};
struct FlowTimer {
    unsigned long long acc = 0;
    unsigned long long t0 = 0;
    __device__ __forceinline__ void start(bool on) { if (on) t0 = clock64(); }
    __device__ __forceinline__ void stop(bool on) { if (on) acc += clock64() - t0; }
};

// ---------------------------------------------------------------- flags
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// spin until *p >= target (a unit earlier in the global order will raise it), then order
// this thread's later async-proxy (TMA) reads after what the acquire made visible
__device__ __forceinline__ void flow_wait(const int *p, int target) {
    if (ld_acquire(p) < target) {
        do {
            __nanosleep(128);
        } while (ld_acquire(p) < target);
    }
    fence_proxy_async_global();
}
__device__ __forceinline__ uint4 ld_cg_u4(const void *p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void tma_store_2d_hint(const void *tmap, const void *src_smem, int c0,
                                                  int c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
            tmap),
        "r"(c0), "r"(c1), "r"(smem_u32(src_smem)), "l"(policy)
        : "memory");
}

// ---------------------------------------------------------------- the unit streams
// Pairs (q, t) in the order s = q + t ascending, then t ascending (q descending); each pair
// has `per` units.  A CTA walks units first, first + step, ... of that order.
struct FlowCursor {
    int q, t, sub;
    int64_t pidx;   // pair index (end: np * ntiles)
    // pairs in the order: s = q + t / G ascending, then q descending, then t ascending
    // (tile groups of G tiles move through the passes as a wavefront)
    int G, ng;
    __device__ __forceinline__ void next_pair(int np, int ntiles) {
        ++pidx;
        const int g = t / G;
        const int tl = t - g * G;
        const int gsz = min(G, ntiles - g * G);
        if (tl + 1 < gsz) {
            ++t;
            return;
        }
        const int s = q + g;
        if (q > 0 && g + 1 < ng) {   // next group of the same diagonal, one pass lower
            --q;
            t = (g + 1) * G;
            return;
        }
        const int s1 = s + 1;
        q = s1 < np - 1 ? s1 : np - 1;
        t = (s1 - q) * G;
    }
    __device__ __forceinline__ void init(int first, int per, int np, int ntiles, int G_) {
        G = G_;
        ng = (ntiles + G - 1) / G;
        q = 0;
        t = 0;
        pidx = 0;
        sub = first;
        while (sub >= per && pidx < static_cast<int64_t>(np) * ntiles) {
            sub -= per;
            next_pair(np, ntiles);
        }
    }
    __device__ __forceinline__ void advance(int step, int per, int np, int ntiles) {
        sub += step;
        while (sub >= per && pidx < static_cast<int64_t>(np) * ntiles) {
            sub -= per;
            next_pair(np, ntiles);
        }
    }
    __device__ __forceinline__ bool valid(int np, int ntiles) const {
        return pidx < static_cast<int64_t>(np) * ntiles;
    }
};

template <typename Fn>
__device__ __forceinline__ void flow_for_units(const FlowArgs &A, int first, int step, int per,
                                               Fn &&fn) {
    FlowCursor c;
    c.init(first, per, A.np, A.ntiles, A.G);
    while (c.valid(A.np, A.ntiles)) {
        fn(c.q, c.t, c.sub);
        c.advance(step, per, A.np, A.ntiles);
    }
}

// K range [klo, khi) of project unit kc of pass q (empty when klo >= khi)
__device__ __forceinline__ void flow_krange(const FlowArgs &A, const FlowPass &ps, int kc, int &klo,
                                            int &khi) {
    const int nk = (A.n + 31) / 32;
    const int span = nk - ps.ks0;
    const int per = (span + A.nkc - 1) / A.nkc;
    klo = ps.ks0 + kc * per;
    khi = klo + per < nk ? klo + per : nk;
}

// ---------------------------------------------------------------- project role (K5a body)
__device__ __forceinline__ void flow_project(const FlowArgs &A, unsigned char *smem) {
    const int kwmax = A.kwmax;
    const int nraw = A.nraw;
    const int cvb = 16384 + 128 * kwmax;
    unsigned char *conv = smem + nraw * kRawBytes;
    Bars1 *bars = reinterpret_cast<Bars1 *>(conv + kStages1 * cvb);
    auto rawX = [&](int s) { return smem + s * kRawBytes; };
    auto Xhi = [&](int s) { return conv + s * cvb; };
    auto Xlo = [&](int s) { return conv + s * cvb + 8192; };
    auto Whi = [&](int s) { return conv + s * cvb + 16384; };
    auto Wlo = [&](int s, int kw) { return conv + s * cvb + 16384 + 64 * kw; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int first = blockIdx.x, step = A.P, per = A.nkc;
    const bool dbg = A.tl != nullptr;
    unsigned long long *tl = dbg ? A.tl + static_cast<int64_t>(blockIdx.x) * 16 : nullptr;
    FlowTimer t_a, t_b, t_c;
    unsigned long long nunits = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nraw; ++s) {
            mbar_init(&bars->rfull[s], 1);
            mbar_init(&bars->rempty[s], 256);
        }
        for (int s = 0; s < kStages1; ++s) {
            mbar_init(&bars->wfull[s], 1);
            mbar_init(&bars->cfull[s], 256);
            mbar_init(&bars->cempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 128);
        }
        fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc<512>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;

    if (warp == 0) {
        if (lane == 0) {
            tc::prefetch_tmap(&A.mXp);
            tc::prefetch_tmap(&A.mYp);
            // re-read by the update role from L2
            const uint64_t pol = (A.pol & 1) ? policy_evict_last() : policy_evict_normal();
            int s = 0;
            uint32_t ph = 0;
            flow_for_units(A, first, step, per, [&](int q, int t, int kc) {
                const FlowPass &ps = A.pass[q];
                int klo, khi;
                flow_krange(A, ps, kc, klo, khi);
                if (klo >= khi) return;
                // dependencies: the previous pass of this tile has stored all its rows, or
                // (first pass) tile t - D has left the program (the L2 window)
                t_a.start(dbg);
                if (q > 0)
                    flow_wait(A.udone + static_cast<int64_t>(q - 1) * A.ntiles + t, A.pass[q - 1].target);
                else if (t >= A.D)
                    flow_wait(A.udone + static_cast<int64_t>(A.np - 1) * A.ntiles + (t - A.D),
                              A.pass[A.np - 1].target);
                t_a.stop(dbg);
                const CUtensorMap *m = q == 0 ? &A.mXp : &A.mYp;
                for (int ks = klo; ks < khi; ++ks) {
                    t_b.start(dbg);
                    mbar_wait(&bars->rempty[s], ph ^ 1u);
                    t_b.stop(dbg);
                    mbar_arrive_expect_tx(&bars->rfull[s], static_cast<uint32_t>(kRawBytes));
                    tc::tma_load_2d_hint(rawX(s), m, ks * 32, t * kTileCols, &bars->rfull[s], pol);
                    if (++s == nraw) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            });
            if (dbg) {
                tl[TL_PDEP] = t_a.acc;
                tl[TL_PRING] = t_b.acc;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            tc::prefetch_tmap(&A.mW[0]);
            tc::prefetch_tmap(&A.mW[1]);
            int s = 0;
            uint32_t ph = 0;
            flow_for_units(A, first, step, per, [&](int q, int, int kc) {
                const FlowPass &ps = A.pass[q];
                int klo, khi;
                flow_krange(A, ps, kc, klo, khi);
                const uint32_t bytes = 128u * static_cast<uint32_t>(ps.kw);
                for (int ks = klo; ks < khi; ++ks) {
                    mbar_wait(&bars->cempty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&bars->wfull[s], bytes);
                    tc::tma_load_2d(Whi(s), &A.mW[ps.wmap], ks * 32, ps.wrow, &bars->wfull[s]);
                    tc::tma_load_2d(Wlo(s, ps.kw), &A.mW[ps.wmap], ks * 32, ps.wrow_lo, &bars->wfull[s]);
                    if (++s == kStages1) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            });
        }
    } else if (warp == 2) {
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0;
        flow_for_units(A, first, step, per, [&](int q, int, int kc) {
            const FlowPass &ps = A.pass[q];
            int klo, khi;
            flow_krange(A, ps, kc, klo, khi);
            const uint32_t idesc = tc::idesc_bf16(128, ps.kw);
            t_b.start(dbg);
            mbar_wait(&bars->acc_empty[a], aph ^ 1u);
            t_b.stop(dbg);
            tc::fence_after_sync();
            const uint32_t d = tbase + static_cast<uint32_t>(a * 256);
            for (int ks = klo; ks < khi; ++ks) {
                t_a.start(dbg);
                mbar_wait(&bars->wfull[s], ph);
                mbar_wait(&bars->cfull[s], ph);
                t_a.stop(dbg);
                tc::fence_after_sync();
                const uint32_t xh = smem_u32(Xhi(s)), xl = smem_u32(Xlo(s));
                const uint32_t wh = smem_u32(Whi(s)), wl = smem_u32(Wlo(s, ps.kw));
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint64_t ah = tc::sdesc_sw64(xh + kk * 32), alo = tc::sdesc_sw64(xl + kk * 32);
                    const uint64_t bh = tc::sdesc_sw64(wh + kk * 32), blo = tc::sdesc_sw64(wl + kk * 32);
                    tc::mma_bf16_w(d, ah, bh, idesc, (ks != klo || kk != 0) ? 1u : 0u);
                    tc::mma_bf16_w(d, ah, blo, idesc, 1u);
                    tc::mma_bf16_w(d, alo, bh, idesc, 1u);
                }
                tc::mma_commit_w(&bars->cempty[s]);
                if (++s == kStages1) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->acc_full[a]);   // (an empty unit arrives at once)
            if (++a == 2) {
                a = 0;
                aph ^= 1u;
            }
        });
        __syncwarp();
        if (dbg && lane == 0) {
            tl[TL_MMA_IN] = t_a.acc;
            tl[TL_MMA_ACC] = t_b.acc;
        }
    } else if (warp < 11) {
        // converters: 256 threads, 4 float4 each per K step (fp32 X tile -> bf16 hi/lo)
        const int ct = threadIdx.x - 96;
        int rs = 0, cs = 0;
        uint32_t rph = 0, cph = 0;
        flow_for_units(A, first, step, per, [&](int q, int, int kc) {
            const FlowPass &ps = A.pass[q];
            int klo, khi;
            flow_krange(A, ps, kc, klo, khi);
            for (int ks = klo; ks < khi; ++ks) {
                t_a.start(dbg);
                mbar_wait(&bars->rfull[rs], rph);
                t_a.stop(dbg);
                const uint32_t raw = smem_u32(rawX(rs));
                float4 v[4];
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) v[qq] = tc::lds128(raw + (ct + 256 * qq) * 16);
                if (ps.dscale) {   // NEXT-f1 right factor: project D X
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        const int r = ks * 32 + ((ct + 256 * qq) & 7) * 4;
                        if (r < A.n) {
                            const float4 dv = *reinterpret_cast<const float4 *>(ps.dscale + r);
                            v[qq].x *= dv.x;
                            v[qq].y *= dv.y;
                            v[qq].z *= dv.z;
                            v[qq].w *= dv.w;
                        }
                    }
                }
                t_b.start(dbg);
                mbar_wait(&bars->cempty[cs], cph ^ 1u);
                t_b.stop(dbg);
                const uint32_t xh = smem_u32(Xhi(cs)), xl = smem_u32(Xlo(cs));
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const int idx = ct + 256 * qq;
                    const int r = idx >> 3, c4 = idx & 7;
                    uint2 Hh, Ll;
                    tc::split2(v[qq].x, v[qq].y, Hh.x, Ll.x);
                    tc::split2(v[qq].z, v[qq].w, Hh.y, Ll.y);
                    const uint32_t off = tc::sw64_off(r, c4 >> 1) + (c4 & 1) * 8;
                    tc::sts64(xh + off, Hh.x, Hh.y);
                    tc::sts64(xl + off, Ll.x, Ll.y);
                }
                fence_proxy_async_smem();
                tc::mbar_arrive(&bars->rempty[rs]);
                tc::mbar_arrive(&bars->cfull[cs]);
                if (++rs == nraw) {
                    rs = 0;
                    rph ^= 1u;
                }
                if (++cs == kStages1) {
                    cs = 0;
                    cph ^= 1u;
                }
            }
        });
        if (dbg && ct == 0) {
            tl[TL_CV_IN] = t_a.acc;
            tl[TL_CV_OUT] = t_b.acc;
        }
    } else if (warp < 15) {
        // epilogue: TMEM lane quarter qd = warp % 4 = columns j of the tile
        const int qd = warp & 3;
        const int jl = qd * 32 + lane;
        int a = 0;
        uint32_t aph = 0;
        const int nkc = A.nkc;
        const int64_t lo_rows = static_cast<int64_t>(A.D) * kTileCols;
        flow_for_units(A, first, step, per, [&](int q, int t, int kc) {
            const FlowPass &ps = A.pass[q];
            int klo, khi;
            flow_krange(A, ps, kc, klo, khi);
            const bool empty = klo >= khi;
            const int slot = t % A.D;
            const int nsl = ps.kw / 16;   // 16-column groups of G
            t_a.start(dbg);
            mbar_wait(&bars->acc_full[a], aph);
            t_a.stop(dbg);
            ++nunits;
            t_c.start(dbg);
            tc::fence_after_sync();
            uint16_t *gh = A.ring + (static_cast<int64_t>(slot) * kTileCols + jl) * kwmax;
            uint16_t *gl = A.ring + (lo_rows + static_cast<int64_t>(slot) * kTileCols + jl) * kwmax;
            auto put_g = [&](int c, const float (&v)[16]) {
                uint32_t Hh[8], Ll[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) tc::split2(v[2 * e], v[2 * e + 1], Hh[e], Ll[e]);
                uint4 *ph = reinterpret_cast<uint4 *>(gh + c * 16);
                uint4 *pl = reinterpret_cast<uint4 *>(gl + c * 16);
                ph[0] = make_uint4(Hh[0], Hh[1], Hh[2], Hh[3]);
                ph[1] = make_uint4(Hh[4], Hh[5], Hh[6], Hh[7]);
                pl[0] = make_uint4(Ll[0], Ll[1], Ll[2], Ll[3]);
                pl[1] = make_uint4(Ll[4], Ll[5], Ll[6], Ll[7]);
            };
            auto tload = [&](int c, float (&v)[16]) {
                if (empty) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0.f;
                } else {
                    tc::tmem_ld16(tbase + (static_cast<uint32_t>(qd * 32) << 16) +
                                      static_cast<uint32_t>(a * 256 + c * 16),
                                  v);
                }
            };
            int *gflag = A.gready + static_cast<int64_t>(q) * A.ntiles + t;
            if (nkc == 1) {
                for (int c = 0; c < nsl; ++c) {
                    float v[16];
                    tload(c, v);
                    put_g(c, v);
                }
                tc::fence_before_sync();
                tc::mbar_arrive(&bars->acc_empty[a]);
                __threadfence();
                named_bar_sync(1, 128);
                if (jl == 0) st_release(gflag, 1);
            } else {
                float *mine = A.part + ((static_cast<int64_t>(slot) * nkc + kc) * (kwmax / 16) * kTileCols) * 16;
                for (int c = 0; c < nsl; ++c) {
                    float v[16];
                    tload(c, v);
                    float *dst = mine + (static_cast<int64_t>(c) * kTileCols + jl) * 16;
#pragma unroll
                    for (int e = 0; e < 4; ++e) st_cg4(dst + 4 * e, v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
                }
                tc::fence_before_sync();
                tc::mbar_arrive(&bars->acc_empty[a]);   // the accumulator is free again
                __threadfence();
                named_bar_sync(1, 128);
                if (jl == 0) {
                    const int prev = atomicAdd(A.gcount + static_cast<int64_t>(q) * A.ntiles + t, 1);
                    bars->last = prev == nkc - 1;
                    __threadfence();
                }
                named_bar_sync(1, 128);
                if (bars->last) {
                    t_b.start(dbg);
                    // the last of the tile's nkc units: G = sum of the partials in kc order
                    const float *p0 = A.part + (static_cast<int64_t>(slot) * nkc * (kwmax / 16) * kTileCols) * 16;
                    const int64_t pstride = static_cast<int64_t>(kwmax / 16) * kTileCols * 16;
                    for (int c = 0; c < nsl; ++c) {
                        float v[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = 0.f;
                        for (int k = 0; k < nkc; ++k) {
                            const float *src = p0 + k * pstride + (static_cast<int64_t>(c) * kTileCols + jl) * 16;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float4 pv = ld_cg4(src + 4 * e);
                                v[4 * e] += pv.x;
                                v[4 * e + 1] += pv.y;
                                v[4 * e + 2] += pv.z;
                                v[4 * e + 3] += pv.w;
                            }
                        }
                        put_g(c, v);
                    }
                    __threadfence();
                    named_bar_sync(1, 128);
                    if (jl == 0) st_release(gflag, 1);
                    t_b.stop(dbg);
                }
            }
            t_c.stop(dbg);
            if (++a == 2) {
                a = 0;
                aph ^= 1u;
            }
        });
        if (dbg && jl == 0) {
            tl[TL_EPI_ACC] = t_a.acc;
            tl[TL_EPI_RED] = t_b.acc;
            tl[TL_EPI_BUSY] = t_c.acc;
            tl[TL_UNITS] = nunits;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 2) tc::tmem_free<512>(tbase);
}

// per-unit completion count of the update role: with several passes the next pass reads
// these rows, so the stores must be complete (bulk wait + proxy fence); a one-pass program
// only uses the count for the L2 window, where a retired (issued) store is enough
__device__ __forceinline__ void flow_done(const FlowArgs &A, int q, int t) {
    if (A.np > 1) {
        tc::bulk_wait0();
        fence_proxy_async_global();
        __threadfence();
    }
    atomicAdd(A.udone + static_cast<int64_t>(q) * A.ntiles + t, 1);
}

// update entries: (q, t, row segment) -> row chunks [rlo, rhi), MMA from mlo
__device__ __forceinline__ void flow_rows(const FlowArgs &A, const FlowPass &ps, int seg, int &rlo,
                                          int &rhi, int &mlo) {
    const int nrc = A.n_pad / kRowChunk;
    rlo = seg * A.rseg;
    if (rlo < ps.xrc0) rlo = ps.xrc0;
    rhi = (seg + 1) * A.rseg < nrc ? (seg + 1) * A.rseg : nrc;
    mlo = rlo > ps.rc0 ? rlo : ps.rc0;
}

// ---------------------------------------------------------------- update role, SS (K5b body)
__device__ __forceinline__ void flow_update_ss(const FlowArgs &A, unsigned char *smem) {
    const int nslab_max = A.kwmax / 32;
    const int nxs = A.nxs;
    unsigned char *Ghi = smem;
    unsigned char *Glo = smem + nslab_max * 8192;
    unsigned char *stg = smem + nslab_max * 16384;
    unsigned char *xst = stg + kStages3 * kStage3Bytes;
    Bars3 *bars = reinterpret_cast<Bars3 *>(xst + nxs * kXBoxBytes);
    auto Vhi = [&](int s) { return stg + s * kStage3Bytes; };
    auto Vlo = [&](int s) { return stg + s * kStage3Bytes + 8192; };
    auto Xs = [&](int s) { return reinterpret_cast<float *>(xst + s * kXBoxBytes); };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int first = blockIdx.x - A.P, step = gridDim.x - A.P;
    const bool dbg = A.tl != nullptr;
    unsigned long long *tl = dbg ? A.tl + static_cast<int64_t>(blockIdx.x) * 16 : nullptr;
    FlowTimer t_a, t_b;
    unsigned long long nunits = 0;
    const int per = (A.n_pad / kRowChunk + A.rseg - 1) / A.rseg;
    const int64_t lo_rows = static_cast<int64_t>(A.D) * kTileCols;
    if (threadIdx.x == 0) {
        mbar_init(&bars->gfull, 1);
        mbar_init(&bars->gempty, 1);
        for (int s = 0; s < kStages3; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int s = 0; s < nxs; ++s) {
            mbar_init(&bars->xfull[s], 1);
            mbar_init(&bars->xempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 512);
        }
        fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<256>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;

    if (warp == 0) {
        if (lane == 0) {
            tc::prefetch_tmap(&A.mG);
            for (int v = 0; v < 3; ++v) tc::prefetch_tmap(&A.mV[v]);
            int s = 0;
            uint32_t ph = 0, gph = 0;
            flow_for_units(A, first, step, per, [&](int q, int t, int seg) {
                const FlowPass &ps = A.pass[q];
                int rlo, rhi, mlo;
                flow_rows(A, ps, seg, rlo, rhi, mlo);
                if (mlo >= rhi) return;   // copy-only (or empty) entry: no G, no V
                const int nslab = ps.kw / 32;
                t_a.start(dbg);
                flow_wait(A.gready + static_cast<int64_t>(q) * A.ntiles + t, 1);
                t_a.stop(dbg);
                t_b.start(dbg);
                mbar_wait(&bars->gempty, gph ^ 1u);
                t_b.stop(dbg);
                mbar_arrive_expect_tx(&bars->gfull, static_cast<uint32_t>(nslab) * 16384u);
                const int slot = t % A.D;
                for (int c = 0; c < nslab; ++c) {
                    tc::tma_load_2d(Ghi + c * 8192, &A.mG, c * 32, slot * kTileCols, &bars->gfull);
                    tc::tma_load_2d(Glo + c * 8192, &A.mG, c * 32,
                                    static_cast<int>(lo_rows) + slot * kTileCols, &bars->gfull);
                }
                gph ^= 1u;
                const CUtensorMap *mv = &A.mV[ps.vmap];
                for (int rc = mlo; rc < rhi; ++rc) {
                    for (int c = 0; c < nslab; ++c) {
                        t_b.start(dbg);
                        mbar_wait(&bars->empty[s], ph ^ 1u);
                        t_b.stop(dbg);
                        mbar_arrive_expect_tx(&bars->full[s], static_cast<uint32_t>(kStage3Bytes));
                        tc::tma_load_2d(Vhi(s), mv, c * 32, ps.vrow_hi + rc * kRowChunk, &bars->full[s]);
                        tc::tma_load_2d(Vlo(s), mv, c * 32, ps.vrow_lo + rc * kRowChunk, &bars->full[s]);
                        if (++s == kStages3) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
            if (dbg) {
                tl[TL_PDEP] = t_a.acc;
                tl[TL_PRING] = t_b.acc;
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = tc::idesc_bf16(kRowChunk, kTileCols);
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0, gph = 0;
        const uint32_t gh0 = smem_u32(Ghi), gl0 = smem_u32(Glo);
        flow_for_units(A, first, step, per, [&](int q, int, int seg) {
            const FlowPass &ps = A.pass[q];
            int rlo, rhi, mlo;
            flow_rows(A, ps, seg, rlo, rhi, mlo);
            if (mlo >= rhi) return;
            const int nslab = ps.kw / 32;
            t_a.start(dbg);
            mbar_wait(&bars->gfull, gph);
            t_a.stop(dbg);
            gph ^= 1u;
            tc::fence_after_sync();
            for (int rc = mlo; rc < rhi; ++rc) {
                t_b.start(dbg);
                mbar_wait(&bars->acc_empty[a], aph ^ 1u);
                t_b.stop(dbg);
                tc::fence_after_sync();
                const uint32_t d = tbase + static_cast<uint32_t>(a * kTileCols);
                for (int c = 0; c < nslab; ++c) {
                    t_a.start(dbg);
                    mbar_wait(&bars->full[s], ph);
                    t_a.stop(dbg);
                    tc::fence_after_sync();
                    const uint32_t vh = smem_u32(Vhi(s)), vl = smem_u32(Vlo(s));
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint64_t ah = tc::sdesc_sw64(vh + kk * 32), alo = tc::sdesc_sw64(vl + kk * 32);
                        const uint64_t bh = tc::sdesc_sw64(gh0 + c * 8192 + kk * 32);
                        const uint64_t blo = tc::sdesc_sw64(gl0 + c * 8192 + kk * 32);
                        tc::mma_bf16_w(d, ah, bh, idesc, (c | kk) != 0);
                        tc::mma_bf16_w(d, ah, blo, idesc, 1u);
                        tc::mma_bf16_w(d, alo, bh, idesc, 1u);
                    }
                    tc::mma_commit_w(&bars->empty[s]);
                    if (++s == kStages3) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc::mma_commit_w(&bars->acc_full[a]);
                if (++a == 2) {
                    a = 0;
                    aph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->gempty);
        });
        __syncwarp();
        if (dbg && lane == 0) {
            tl[TL_MMA_IN] = t_a.acc;
            tl[TL_MMA_ACC] = t_b.acc;
        }
    } else if (warp == 2) {
        if (lane == 0) {
            tc::prefetch_tmap(&A.mXu);
            tc::prefetch_tmap(&A.mYu);
            const uint64_t pol = (A.pol & 2) ? policy_evict_first() : policy_evict_normal();
            int s = 0;
            uint32_t ph = 0;
            flow_for_units(A, first, step, per, [&](int q, int t, int seg) {
                const FlowPass &ps = A.pass[q];
                int rlo, rhi, mlo;
                flow_rows(A, ps, seg, rlo, rhi, mlo);
                if (rlo >= rhi) return;
                // the tile's G is ready, hence its projection (and the previous pass) is done
                t_a.start(dbg);
                flow_wait(A.gready + static_cast<int64_t>(q) * A.ntiles + t, 1);
                t_a.stop(dbg);
                const CUtensorMap *m = q == 0 ? &A.mXu : &A.mYu;
                for (int rc = rlo; rc < rhi; ++rc) {
                    for (int cb = 0; cb < kTileCols / kXBoxCols; ++cb) {
                        t_b.start(dbg);
                        mbar_wait(&bars->xempty[s], ph ^ 1u);
                        t_b.stop(dbg);
                        mbar_arrive_expect_tx(&bars->xfull[s], static_cast<uint32_t>(kXBoxBytes));
                        tc::tma_load_2d_hint(Xs(s), m, rc * kRowChunk, t * kTileCols + cb * kXBoxCols,
                                             &bars->xfull[s], pol);
                        if (++s == nxs) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
            if (dbg) {
                tl[TL_UDEP] = t_a.acc;
                tl[TL_CV_OUT] = t_b.acc;
            }
        }
    } else if (warp >= 4) {
        const int qd = warp & 3, grp = (warp - 4) >> 2;
        const int r_in = qd * 32 + lane;
        const bool storer = qd == 0 && lane == 0;
        const uint64_t spol = policy_evict_first();
        int a = 0;
        uint32_t aph = 0;
        constexpr int kBoxes = kTileCols / kXBoxCols;
        int64_t seq = 0;
        flow_for_units(A, first, step, per, [&](int q, int t, int seg) {
            const FlowPass &ps = A.pass[q];
            int rlo, rhi, mlo;
            flow_rows(A, ps, seg, rlo, rhi, mlo);
            for (int rc = rlo; rc < rhi; ++rc, seq += kBoxes) {
                const bool mma_rc = rc >= mlo;
                ++nunits;
                if (mma_rc) {
                    t_a.start(dbg);
                    mbar_wait(&bars->acc_full[a], aph);
                    t_a.stop(dbg);
                    tc::fence_after_sync();
                }
                const int r = rc * kRowChunk + r_in;
                const float lr = (ps.pre && r < A.n) ? ps.pre[r] : 1.f;
                const float pr = (ps.post && r < A.n) ? ps.post[r] : 1.f;
#pragma unroll
                for (int k = 0; k < kBoxes / 4; ++k) {
                    const int cb = grp + 4 * k;
                    const int64_t sq = seq + cb;
                    const int s = static_cast<int>(sq % nxs);
                    t_b.start(dbg);
                    mbar_wait(&bars->xfull[s], static_cast<uint32_t>((sq / nxs) & 1));
                    t_b.stop(dbg);
                    const uint32_t xs = smem_u32(Xs(s)) + static_cast<uint32_t>(r_in) * 4u;
                    float v[16];
                    if (mma_rc) {
                        tc::tmem_ld16(tbase + (static_cast<uint32_t>(qd * 32) << 16) +
                                          static_cast<uint32_t>(a * kTileCols + cb * kXBoxCols),
                                      v);
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    }
#pragma unroll
                    for (int e = 0; e < kXBoxCols; ++e) {
                        const uint32_t ad = xs + e * kRowChunk * 4;
                        sts_f32(ad, pr * fmaf(lr, lds_f32(ad), -v[e]));
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1 + grp, 128);
                    if (storer) {
                        tma_store_2d_hint(&A.mYu, Xs(s), rc * kRowChunk, t * kTileCols + cb * kXBoxCols, spol);
                        tc::bulk_commit();
                        tc::bulk_wait_read0();   // the box may be refilled once TMA has read it
                        tc::mbar_arrive(&bars->xempty[s]);
                    }
                }
                if (mma_rc) {
                    tc::fence_before_sync();
                    tc::mbar_arrive(&bars->acc_empty[a]);
                    if (++a == 2) {
                        a = 0;
                        aph ^= 1u;
                    }
                }
                if (storer) flow_done(A, q, t);
            }
        });
        if (storer) tc::bulk_wait0();
        if (dbg && warp == 4 && lane == 0) {
            tl[TL_EPI_ACC] = t_a.acc;
            tl[TL_EPI_X] = t_b.acc;
            tl[TL_UNITS] = nunits;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_free<256>(tbase);
}

// ---------------------------------------------------------------- update role, TS (K5b-TS body)
__device__ __forceinline__ void flow_update_ts(const FlowArgs &A, unsigned char *smem) {
    unsigned char *stg = smem;
    unsigned char *xst = stg + kVS2 * kStage3Bytes;
    Bars4 *bars = reinterpret_cast<Bars4 *>(xst + kXS2 * kXB2Bytes);
    auto Vhi = [&](int s) { return stg + s * kStage3Bytes; };
    auto Vlo = [&](int s) { return stg + s * kStage3Bytes + 8192; };
    auto Xs = [&](int s) { return xst + s * kXB2Bytes; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int first = blockIdx.x - A.P, step = gridDim.x - A.P;
    const int per = (A.n_pad / kRowChunk + A.rseg - 1) / A.rseg;
    const int64_t lo_rows = static_cast<int64_t>(A.D) * kTileCols;
    if (threadIdx.x == 0) {
        mbar_init(&bars->gfull, 512);
        mbar_init(&bars->gempty, 1);
        for (int s = 0; s < kVS2; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int s = 0; s < kXS2; ++s) {
            mbar_init(&bars->xfull[s], 1);
            mbar_init(&bars->xempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 512);
        }
        fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<512>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;

    if (warp == 0) {
        if (lane == 0) {
            for (int v = 0; v < 3; ++v) tc::prefetch_tmap(&A.mV[v]);
            int s = 0;
            uint32_t ph = 0;
            flow_for_units(A, first, step, per, [&](int q, int, int seg) {
                const FlowPass &ps = A.pass[q];
                int rlo, rhi, mlo;
                flow_rows(A, ps, seg, rlo, rhi, mlo);
                const int nslab = ps.kw / 32;
                const CUtensorMap *mv = &A.mV[ps.vmap];
                for (int rc = mlo; rc < rhi; ++rc) {
                    for (int c = 0; c < nslab; ++c) {
                        mbar_wait(&bars->empty[s], ph ^ 1u);
                        mbar_arrive_expect_tx(&bars->full[s], static_cast<uint32_t>(kStage3Bytes));
                        tc::tma_load_2d(Vhi(s), mv, c * 32, ps.vrow_hi + rc * kRowChunk, &bars->full[s]);
                        tc::tma_load_2d(Vlo(s), mv, c * 32, ps.vrow_lo + rc * kRowChunk, &bars->full[s]);
                        if (++s == kVS2) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
        }
    } else if (warp == 1) {
        const uint32_t idesc = tc::idesc_bf16(kTileCols, kRowChunk);
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0, gph = 0;
        flow_for_units(A, first, step, per, [&](int q, int, int seg) {
            const FlowPass &ps = A.pass[q];
            int rlo, rhi, mlo;
            flow_rows(A, ps, seg, rlo, rhi, mlo);
            if (mlo >= rhi) return;
            const int nslab = ps.kw / 32;
            mbar_wait(&bars->gfull, gph);   // this entry's G is in TMEM
            gph ^= 1u;
            tc::fence_after_sync();
            for (int rc = mlo; rc < rhi; ++rc) {
                mbar_wait(&bars->acc_empty[a], aph ^ 1u);
                tc::fence_after_sync();
                const uint32_t d = tbase + 256u + static_cast<uint32_t>(a * kRowChunk);
                for (int c = 0; c < nslab; ++c) {
                    mbar_wait(&bars->full[s], ph);
                    tc::fence_after_sync();
                    const uint32_t vh = smem_u32(Vhi(s)), vl = smem_u32(Vlo(s));
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint64_t bh = tc::sdesc_sw64(vh + kk * 32), bl = tc::sdesc_sw64(vl + kk * 32);
                        const uint32_t ah = tbase + static_cast<uint32_t>(c * 16 + kk * 8);
                        const uint32_t alo = ah + 128u;
                        tc::mma_bf16_ts_w(d, ah, bh, idesc, (c | kk) != 0);
                        tc::mma_bf16_ts_w(d, ah, bl, idesc, 1u);
                        tc::mma_bf16_ts_w(d, alo, bh, idesc, 1u);
                    }
                    tc::mma_commit_w(&bars->empty[s]);
                    if (++s == kVS2) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc::mma_commit_w(&bars->acc_full[a]);
                if (++a == 2) {
                    a = 0;
                    aph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->gempty);   // G may be replaced once these MMAs finish
        });
        __syncwarp();
    } else if (warp == 2) {
        if (lane == 0) {
            tc::prefetch_tmap(&A.mXu);
            tc::prefetch_tmap(&A.mYu);
            const uint64_t pol = (A.pol & 2) ? policy_evict_first() : policy_evict_normal();
            int s = 0;
            uint32_t ph = 0;
            flow_for_units(A, first, step, per, [&](int q, int t, int seg) {
                const FlowPass &ps = A.pass[q];
                int rlo, rhi, mlo;
                flow_rows(A, ps, seg, rlo, rhi, mlo);
                if (rlo >= rhi) return;
                flow_wait(A.gready + static_cast<int64_t>(q) * A.ntiles + t, 1);
                const CUtensorMap *m = q == 0 ? &A.mXu : &A.mYu;
                for (int rc = rlo; rc < rhi; ++rc) {
                    for (int g = 0; g < 4; ++g) {
                        mbar_wait(&bars->xempty[s], ph ^ 1u);
                        mbar_arrive_expect_tx(&bars->xfull[s], static_cast<uint32_t>(kXB2Bytes));
                        tc::tma_load_2d_hint(Xs(s), m, rc * kRowChunk + g * 32, t * kTileCols,
                                             &bars->xfull[s], pol);
                        if (++s == kXS2) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
        }
    } else if (warp >= 4) {
        const int qd = warp & 3, g = (warp - 4) >> 2;
        const int j = qd * 32 + lane;                    // column within the tile (TMEM lane)
        const uint32_t tlane = static_cast<uint32_t>(qd * 32) << 16;
        const bool storer = qd == 0 && lane == 0;
        const uint64_t spol = policy_evict_first();
        int a = 0;
        uint32_t aph = 0, gph = 0;
        int64_t seq = 0;
        flow_for_units(A, first, step, per, [&](int q, int t, int seg) {
            const FlowPass &ps = A.pass[q];
            int rlo, rhi, mlo;
            flow_rows(A, ps, seg, rlo, rhi, mlo);
            if (mlo < rhi) {
                // stage this entry's G (columns = TMEM lanes) once it is published and the
                // previous entry's MMAs are done with TMEM: one thread polls the flag
                if (warp == 4 && lane == 0) flow_wait(A.gready + static_cast<int64_t>(q) * A.ntiles + t, 1);
                named_bar_sync(6, 512);
                mbar_wait(&bars->gempty, gph ^ 1u);
                gph ^= 1u;
                tc::fence_after_sync();
                const int slot = t % A.D;
                const int wq = ps.kw / 4;                   // words per group (multiple of 8)
                const int half = g >> 1;                    // groups 0,1: hi; 2,3: lo
                const int w0 = (g & 1) * wq;                // first word within the half
                const uint16_t *src16 = A.ring + ((half ? lo_rows : 0) + static_cast<int64_t>(slot) * kTileCols + j) *
                                                     A.kwmax + 2 * w0;
                uint4 u[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    u[i] = make_uint4(0u, 0u, 0u, 0u);
                    if (i < wq / 4) u[i] = ld_cg_u4(src16 + 8 * i);
                }
#pragma unroll
                for (int i = 0; i < 16; i += 2)
                    if (i < wq / 4)
                        tc::tmem_st8(tbase + tlane + static_cast<uint32_t>(half * 128 + w0 + 4 * i), u[i], u[i + 1]);
                tc::tmem_wait_st();
                tc::fence_before_sync();
                tc::mbar_arrive(&bars->gfull);
            }
            for (int rc = rlo; rc < rhi; ++rc, seq += 4) {
                const bool mma_rc = rc >= mlo;
                float v[32];
                if (mma_rc) {
                    mbar_wait(&bars->acc_full[a], aph);
                    tc::fence_after_sync();
                    tc::tmem_ld32(tbase + tlane + 256u + static_cast<uint32_t>(a * kRowChunk + g * 32), v);
                    tc::fence_before_sync();
                    tc::mbar_arrive(&bars->acc_empty[a]);
                    if (++a == 2) {
                        a = 0;
                        aph ^= 1u;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
                const int r0 = rc * kRowChunk + g * 32;
                const int64_t sq = seq + g;
                const int s = static_cast<int>(sq % kXS2);
                mbar_wait(&bars->xfull[s], static_cast<uint32_t>((sq / kXS2) & 1));
                const uint32_t xs = smem_u32(Xs(s)) + static_cast<uint32_t>(j) * 128u;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t ad = xs + static_cast<uint32_t>((c ^ (j & 7)) << 4);
                    float4 x4 = tc::lds128(ad);
                    float lr[4] = {1.f, 1.f, 1.f, 1.f}, pr[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int r = r0 + 4 * c + e;
                        if (ps.pre && r < A.n) lr[e] = __ldg(ps.pre + r);
                        if (ps.post && r < A.n) pr[e] = __ldg(ps.post + r);
                    }
                    x4.x = pr[0] * fmaf(lr[0], x4.x, -v[4 * c]);
                    x4.y = pr[1] * fmaf(lr[1], x4.y, -v[4 * c + 1]);
                    x4.z = pr[2] * fmaf(lr[2], x4.z, -v[4 * c + 2]);
                    x4.w = pr[3] * fmaf(lr[3], x4.w, -v[4 * c + 3]);
                    tc::sts128(ad, x4);
                }
                fence_proxy_async_smem();
                named_bar_sync(1 + g, 128);
                if (storer) {
                    tma_store_2d_hint(&A.mYu, Xs(s), r0, t * kTileCols, spol);
                    tc::bulk_commit();
                    tc::bulk_wait_read0();
                    tc::mbar_arrive(&bars->xempty[s]);
                    flow_done(A, q, t);
                }
            }
        });
        if (storer) tc::bulk_wait0();
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_free<512>(tbase);
}

__global__ void __launch_bounds__(640, 1) wy_flow_kernel(const __grid_constant__ FlowArgs A) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const unsigned long long t0 = clock64();
    if (static_cast<int>(blockIdx.x) < A.P)
        flow_project(A, smem);
    else if (A.ts)
        flow_update_ts(A, smem);
    else
        flow_update_ss(A, smem);
    if (A.tl && threadIdx.x == 0) {
        A.tl[static_cast<int64_t>(blockIdx.x) * 16 + TL_ROLE] = static_cast<int>(blockIdx.x) < A.P ? 0 : 1;
        A.tl[static_cast<int64_t>(blockIdx.x) * 16 + TL_TOTAL] = clock64() - t0;
    }
}
