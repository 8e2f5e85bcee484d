// dist_api.cuh -- knng_build_sharded: GNND on every rank's shard, then the
// log-depth GGM tree with every level merged by ALL ranks of its group
// (SURVEY.md section 8(e) stage B).
//
// Included by knng_api.cu inside its anonymous namespace (uses Ctx, Run,
// make_layout, get_workspace).  Ids: the tree numbers every merge from its
// group's first row (D36), so at level l rank r (group g0 = r & ~(2^(l+1)-1))
// owns the merge ids [(r - g0) n_l, (r - g0 + 1) n_l) and A = the group's
// first half.  Between levels the lists hold global ids.
#pragma once
// (comm.cuh, dist_kernels.cuh and <functional> are included by knng_api.cu)

// growable stream-ordered device buffer
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaStream_t st = nullptr;
    explicit DevBuf(cudaStream_t s) : st(s) {}
    DevBuf(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    bool ensure(size_t bytes) {
        if (bytes <= cap) return true;
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        cap = 0;
        bytes = align_up(bytes + bytes / 8);
        if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        cap = bytes;
        return true;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t bytes) {
        if (cudaMallocHost(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
    }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

struct Sharded {
    Comm& C;
    Ctx& c;
    std::string err;
    knng_status code = KNNG_OK;
    PinnedBuf pin{64 * 1024};

    Sharded(Comm& comm, Ctx& ctx) : C(comm), c(ctx) {}

    bool failed() const { return code != KNNG_OK || c.err != cudaSuccess; }
    bool set_err(knng_status s, const std::string& m) {
        if (code == KNNG_OK) {
            code = s;
            err = m;
        }
        return false;
    }
    bool sync() {
        const cudaError_t e = cudaStreamSynchronize(c.stream);
        if (e != cudaSuccess && c.err == cudaSuccess) {
            c.err = e;
            c.err_where = "sharded build";
        }
        return !failed();
    }
    // exchange with the peers in [lo, hi) (this rank's own part is the caller's)
    bool xchg(int lo, int hi, const std::function<Xfer(int)>& snd, const std::function<Xfer(int)>& rcv) {
        if (failed()) return false;
        std::vector<Xfer> s, r;
        for (int q = lo; q < hi; ++q) {
            if (q == C.rank) continue;
            s.push_back(snd(q));
            r.push_back(rcv(q));
        }
        const std::string e = C.exchange(s, r, c.stream);
        if (!e.empty()) return set_err(KNNG_E_NCCL, e);
        return true;
    }
};

knng_status run_sharded(Comm& C, const void* Xloc, int64_t nl, int64_t goff, int64_t ntot, knng_dtype dt, int d,
                        int k, knng_metric metric, int iters, int merge_iters, const int32_t* level_iters, int p,
                        uint64_t seed, uint32_t* out_ids, float* out_dists, cudaStream_t stream) {
    const int P = C.world, r = C.rank;
    int levels = 0;
    while ((1 << levels) < P) ++levels;
    Ctx c;
    c.stream = stream;
    c.timing = g_timing.load() != 0;
    Sharded Z(C, c);
    int64_t* hp = static_cast<int64_t*>(Z.pin.p);
    if (!hp) return fail(KNNG_E_NOMEM, "cannot allocate pinned host memory");

    // ---- every rank checks that all ranks called with the same parameters
    DevBuf pbuf(stream);
    constexpr int NPAR = 16;
    if (!pbuf.ensure(static_cast<size_t>(P) * NPAR * 8)) return fail(KNNG_E_NOMEM, "device allocation failed");
    {
        int64_t mine[NPAR] = {nl, ntot, dt, d, k, metric, iters, merge_iters, p, static_cast<int64_t>(seed), P,
                              goff - static_cast<int64_t>(r) * nl, 0, 0, 0, 0};
        for (int l = 0; l < levels; ++l) mine[12 + (l < 4 ? l : 3)] += level_iters ? level_iters[l] : merge_iters;
        int64_t* dp = pbuf.as<int64_t>();
        cudaMemcpyAsync(dp + static_cast<size_t>(r) * NPAR, mine, sizeof(mine), cudaMemcpyHostToDevice, stream);
        Z.xchg(0, P, [&](int q) { return Xfer{q, dp + static_cast<size_t>(r) * NPAR, NPAR * 8}; },
               [&](int q) { return Xfer{q, dp + static_cast<size_t>(q) * NPAR, NPAR * 8}; });
        cudaMemcpyAsync(hp, dp, static_cast<size_t>(P) * NPAR * 8, cudaMemcpyDeviceToHost, stream);
        if (!Z.sync()) return Z.code ? fail(Z.code, "%s", Z.err.c_str()) : c.finish();
        for (int q = 0; q < P; ++q)
            for (int j = 0; j < NPAR; ++j)
                if (hp[q * NPAR + j] != mine[j])
                    return fail(KNNG_E_USAGE, "rank %d called knng_build_sharded with different parameters "
                                "(or a global_offset other than rank * n_local)", q);
    }

    // ---- replicated vector store, indexed by global id (filled level by level)
    const bool cosine = metric == KNNG_COSINE;
    knng_dtype dte = dt;  // element type of the store (exact-u8 decision below)
    DevBuf flag(stream);
    if (!flag.ensure(static_cast<size_t>(P) * 4 + 256)) return fail(KNNG_E_NOMEM, "device allocation failed");
    int* fl = flag.as<int>();
    cudaMemsetAsync(fl, 0, static_cast<size_t>(P) * 4 + 256, stream);
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // flags of every rank: bit 0 = some value is not an integer in [0, 255]
    // (D35), bit 1 = a zero row under cosine (D6); agreed on by all ranks
    const size_t rowf = static_cast<size_t>(d) * 4;
    DevBuf Xall(stream);
    const bool try_u8 = metric == KNNG_L2SQ && dt == KNNG_F32 && d <= 258 && g_opt_exact_u8.load();
    const bool chi2 = metric == KNNG_CHI2;
    if (!Xall.ensure(static_cast<size_t>(ntot) * (dt == KNNG_U8 && !cosine && !chi2 ? d : rowf)))
        return fail(KNNG_E_NOMEM, "cannot allocate the vector store");
    char* Xs = Xall.as<char>();
    if (cosine) {
        cudaMemsetAsync(fl + P, 0, 4, stream);
        c.launch("k_normalize", [&] {
            k_normalize<<<static_cast<int>((nl + 255) / 256), 256, 0, stream>>>(
                static_cast<const float*>(Xloc), nl, d, reinterpret_cast<float*>(Xs + static_cast<size_t>(goff) * rowf), fl + P);
        });
        cudaMemcpyAsync(fl + r, fl + P, 4, cudaMemcpyDeviceToDevice, stream);  // 1 -> bit 0 ...
        c.launch("k_flag_shift", [&] { k_flag_shift<<<1, 1, 0, stream>>>(fl + r); });  // ... -> bit 1
    } else if (chi2 && dt == KNNG_F32) {
        c.launch("k_check_nonneg", [&] {
            k_check_nonneg<<<4 * sms, 256, 0, stream>>>(static_cast<const float*>(Xloc), nl * d, fl + r);
        });
        c.launch("k_flag_shift", [&] { k_flag_shift<<<1, 1, 0, stream>>>(fl + r); });
    } else if (try_u8) {
        c.launch("k_check_u8", [&] {
            k_check_u8<<<4 * sms, 256, 0, stream>>>(static_cast<const float*>(Xloc), nl * d, fl + r);
        });
    }
    Z.xchg(0, P, [&](int q) { return Xfer{q, fl + r, 4}; }, [&](int q) { return Xfer{q, fl + q, 4}; });
    cudaMemcpyAsync(hp, fl, static_cast<size_t>(P) * 4, cudaMemcpyDeviceToHost, stream);
    if (!Z.sync()) return Z.code ? fail(Z.code, "%s", Z.err.c_str()) : c.finish();
    bool all_int = try_u8, zero_row = false;
    for (int q = 0; q < P; ++q) {
        const int f = reinterpret_cast<int*>(hp)[q];
        all_int &= (f & 1) == 0;
        zero_row |= (f & 2) != 0;
    }
    if (zero_row)
        return fail(KNNG_E_DOMAIN, cosine ? "zero vector under the cosine metric"
                                          : "negative value under the chi-square metric");
    if (all_int) dte = KNNG_U8;
    if (chi2) dte = KNNG_F32;  // chi-square runs on float rows (D39)
    g_last_exact_u8 = all_int;
    const size_t esz = (dte == KNNG_U8 && !cosine) ? 1 : 4;  // (chi2: dte is float)
    const size_t rowb = static_cast<size_t>(d) * esz;
    char* Xmine = Xs + static_cast<size_t>(goff) * rowb;
    if (cosine) {
        // normalised rows already in place
    } else if (chi2 && dt == KNNG_U8) {
        c.launch("k_u8_to_f32", [&] {
            k_u8_to_f32<<<4 * sms, 256, 0, stream>>>(static_cast<const uint8_t*>(Xloc), nl * d, reinterpret_cast<float*>(Xmine));
        });
    } else if (dte == KNNG_U8 && dt == KNNG_F32) {
        c.launch("k_to_u8", [&] {
            k_to_u8<<<4 * sms, 256, 0, stream>>>(static_cast<const float*>(Xloc), nl * d, reinterpret_cast<uint8_t*>(Xmine));
        });
    } else {
        cudaMemcpyAsync(Xmine, Xloc, static_cast<size_t>(nl) * rowb, cudaMemcpyDeviceToDevice, stream);
    }

    // ---- 1. GNND on the own shard: seed + rank, then global ids
    DevBuf cur(stream);  // u64 [nl][k]: the own lists, global ids
    if (!cur.ensure(static_cast<size_t>(nl) * k * 8)) return fail(KNNG_E_NOMEM, "device allocation failed");
    {
        DevBuf tids(stream), tdst(stream);
        if (!tids.ensure(static_cast<size_t>(nl) * k * 4) || !tdst.ensure(static_cast<size_t>(nl) * k * 4))
            return fail(KNNG_E_NOMEM, "device allocation failed");
        if (!Z.sync()) return c.finish();
        const knng_status s = knng_build(Xloc, dt, nl, d, k, metric, iters, p, seed + static_cast<uint64_t>(r),
                                         tids.as<uint32_t>(), tdst.as<float>(), nullptr, 0, stream);
        if (s != KNNG_OK) return s;
        std::vector<knng_iter_stats> hist = g_last_stats;
        c.launch("k_to_keys", [&] {
            k_to_keys<<<static_cast<int>((nl * k + 255) / 256), 256, 0, stream>>>(tids.as<uint32_t>(), tdst.as<float>(),
                                                                                   nl * k, goff, cur.as<uint64_t>());
        });
        g_last_stats = hist;
    }
    std::vector<knng_iter_stats> history = g_last_stats;

    // ---- 2. the tree: level l merges groups of 2^(l+1) ranks
    const int cap = 2 * p;
    DevBuf ws_buf(stream), kthall(stream), sqn(stream), fwdrec(stream), recvrec(stream), rpos(stream),
        rsrc(stream), bucket(stream), rec_tgt(stream), rec_key(stream), candout(stream), candin(stream),
        small(stream);
    const Layout L = make_layout(nl, d, k, p, false, true, true, false);
    if (!ws_buf.ensure(L.total) || !kthall.ensure(static_cast<size_t>(ntot) * 8) ||
        !sqn.ensure(static_cast<size_t>(ntot) * 4) || !small.ensure(64 * 1024) ||
        !rec_tgt.ensure(static_cast<size_t>(nl) * 3 * cap * 4 + 256) ||
        !rec_key.ensure(static_cast<size_t>(nl) * 3 * cap * 8 + 256) ||
        !fwdrec.ensure(static_cast<size_t>(nl) * 2 * p * 8 + 256) || !candout.ensure(static_cast<size_t>(nl) * 3 * cap * 16 + 256))
        return fail(KNNG_E_NOMEM, "cannot allocate the distributed-refine state");
    unsigned int* dcnt = small.as<unsigned int>();                                          // [2 P] u32 counts
    unsigned int* rcvc = dcnt + 2 * P;                                                      // [P][2] received counts
    unsigned long long* binoff = reinterpret_cast<unsigned long long*>(small.as<char>() + 16 * 1024);  // [2 P]
    unsigned long long* nrec_d = binoff + 2 * P;

    for (int l = 0; l < levels; ++l) {
        const int gs = 2 << l, g0 = r & ~(gs - 1), h = gs / 2, me = r - g0;
        const int64_t G0 = static_cast<int64_t>(g0) * nl, ngrp = static_cast<int64_t>(gs) * nl;
        const int64_t nA = static_cast<int64_t>(h) * nl, base = static_cast<int64_t>(me) * nl;
        const int mi = level_iters ? level_iters[l] : merge_iters;
        const bool in_a = me < h;
        // vectors of the other half (this rank's half is present from level l-1)
        const int olo = in_a ? g0 + h : g0, ohi = olo + h;
        if (!Z.xchg(g0, g0 + gs,
                    [&](int q) { return Xfer{q, (q >= olo && q < ohi) ? Xmine : nullptr, (q >= olo && q < ohi) ? nl * rowb : 0}; },
                    [&](int q) {
                        const bool o = q >= olo && q < ohi;
                        return Xfer{q, o ? Xs + static_cast<size_t>(q) * nl * rowb : nullptr, o ? nl * rowb : 0};
                    }))
            break;

        Run R(c);
        R.L = L;
        R.D = Dims{nl, d, k, p, cap};
        R.D.base = base;
        R.X = Xs + static_cast<size_t>(G0) * rowb;  // merge ids index the group's rows
        R.dt = dte;
        R.metric = metric;
        R.seed = seed;
        R.boundary = nA;
        R.xrows = ngrp;
        R.sqn_ext = sqn.p;
        R.bind(ws_buf.as<char>(), nullptr);
        R.update = 0;  // the distributed refine files through records (bulk update)
        R.G.lock = nullptr;
        R.G.imask = nullptr;
        if (cosine) R.Xn = reinterpret_cast<const float*>(R.X);
        R.G.kth = kthall.as<uint64_t>() + base;  // merge_sample writes the own slice ...
        R.G.kth_t = kthall.as<uint64_t>();       // ... the joins read the group's
        uint32_t* fpos_buf = R.S.fpos;
        R.S.fpos = nullptr;  // no local reverse counts: records go to the owners
        R.G.rec_tgt = rec_tgt.as<uint32_t>();
        R.G.rec_key = rec_key.as<uint64_t>();
        R.G.rec_cnt = nrec_d;
        R.zero_state();

        // seed (Alg. 3 lines 1-7) from the own lists in merge ids
        uint64_t* reserved = reinterpret_cast<uint64_t*>(R.ws + L.reserved);
        const int64_t tot = nl * k;
        c.launch("k_keys_shift", [&] {
            k_keys_shift<<<static_cast<int>((tot + 255) / 256), 256, 0, stream>>>(cur.as<uint64_t>(), tot, -G0);
        });
        const int grid = R.warps_grid(nl, 8);
        c.launch("k_ggm_seed", [&] {
            if (cosine)
                k_ggm_seed_keys<float, true><<<grid, 256, 256 * 4, stream>>>(nullptr, R.Xn, R.D, nA, ngrp, l, seed,
                                                                          cur.as<uint64_t>(), R.G, reserved);
            else if (chi2)
                k_ggm_seed_keys<float, kMetChi2><<<grid, 256, 256 * 4, stream>>>(static_cast<const float*>(R.X), nullptr, R.D,
                                                                              nA, ngrp, l, seed, cur.as<uint64_t>(), R.G,
                                                                              reserved);
            else if (dte == KNNG_F32)
                k_ggm_seed_keys<float, false><<<grid, 256, 256 * 4, stream>>>(static_cast<const float*>(R.X), nullptr, R.D,
                                                                           nA, ngrp, l, seed, cur.as<uint64_t>(), R.G,
                                                                           reserved);
            else
                k_ggm_seed_keys<uint8_t, false><<<grid, 256, 256 * 4, stream>>>(
                    static_cast<const uint8_t*>(R.X), nullptr, R.D, nA, ngrp, l, seed, cur.as<uint64_t>(), R.G, reserved);
        });

        for (int t = 0; t < mi && !Z.failed(); ++t) {
            const uint32_t tword = 0x80000000u | (static_cast<uint32_t>(l) << 16) | static_cast<uint32_t>(t);
            // (a) bucket merge of t-1 + forward samples of the own nodes
            R.merge_sample(t > 0 ? 1 : 0, 1, t > 0 ? t - 1 : -1);
            // (b) thresholds of the group (D17): own slice -> every member
            uint64_t* ka = kthall.as<uint64_t>();
            Z.xchg(g0, g0 + gs, [&](int q) { return Xfer{q, ka + base, static_cast<size_t>(nl) * 8}; },
                   [&](int q) { return Xfer{q, ka + static_cast<size_t>(q - g0) * nl, static_cast<size_t>(nl) * 8}; });
            // (c) reverse records to the targets' owners
            cudaMemsetAsync(dcnt, 0, static_cast<size_t>(2 * gs) * 4, stream);
            const int64_t items = nl * p;
            c.launch("k_fwd_count", [&] {
                k_fwd_count<<<dim3(static_cast<unsigned>((items + 255) / 256), 2), 256, 0, stream>>>(R.D, R.S, fpos_buf,
                                                                                                     nl, dcnt);
            });
            Z.xchg(g0, g0 + gs, [&](int q) { return Xfer{q, dcnt + 2 * (q - g0), 8}; },
                   [&](int q) { return Xfer{q, rcvc + 2 * (q - g0), 8}; });
            cudaMemcpyAsync(rcvc + 2 * me, dcnt + 2 * me, 8, cudaMemcpyDeviceToDevice, stream);
            unsigned int* hc = reinterpret_cast<unsigned int*>(hp);
            cudaMemcpyAsync(hc, dcnt, static_cast<size_t>(2 * gs) * 4, cudaMemcpyDeviceToHost, stream);
            cudaMemcpyAsync(hc + 2 * gs, rcvc, static_cast<size_t>(2 * gs) * 4, cudaMemcpyDeviceToHost, stream);
            if (!Z.sync()) break;
            std::vector<unsigned long long> sboff(2 * gs), rboff(gs + 1);
            unsigned long long acc = 0;
            for (int j = 0; j < gs; ++j) {
                sboff[2 * j] = acc;
                sboff[2 * j + 1] = acc + hc[2 * j];
                acc += hc[2 * j] + hc[2 * j + 1];
            }
            unsigned long long tf[2] = {0, 0};
            for (int j = 0; j < gs; ++j) {
                rboff[j] = tf[0] + tf[1];
                tf[0] += hc[2 * gs + 2 * j];
                tf[1] += hc[2 * gs + 2 * j + 1];
            }
            const int64_t nrecv = static_cast<int64_t>(tf[0] + tf[1]);
            rboff[gs] = nrecv;
            cudaMemcpyAsync(binoff, sboff.data(), sboff.size() * 8, cudaMemcpyHostToDevice, stream);
            c.launch("k_fwd_scatter", [&] {
                k_fwd_scatter<<<dim3(static_cast<unsigned>((items + 255) / 256), 2), 256, 0, stream>>>(
                    R.D, R.S, fpos_buf, nl, binoff, fwdrec.as<uint2>());
            });
            if (!recvrec.ensure(static_cast<size_t>(nrecv) * 8 + 8) || !rpos.ensure(static_cast<size_t>(nrecv) * 4 + 4)) {
                Z.set_err(KNNG_E_NOMEM, "device allocation failed");
                break;
            }
            uint2* fr = fwdrec.as<uint2>();
            uint2* rr = recvrec.as<uint2>();
            const int meg = me;
            Z.xchg(g0, g0 + gs,
                   [&](int q) {
                       const int j = q - g0;
                       return Xfer{q, fr + sboff[2 * j], static_cast<size_t>(hc[2 * j] + hc[2 * j + 1]) * 8};
                   },
                   [&](int q) {
                       const int j = q - g0;
                       return Xfer{q, rr + rboff[j], static_cast<size_t>(rboff[j + 1] - rboff[j]) * 8};
                   });
            cudaMemcpyAsync(rr + rboff[meg], fr + sboff[2 * meg], static_cast<size_t>(hc[2 * meg] + hc[2 * meg + 1]) * 8,
                            cudaMemcpyDeviceToDevice, stream);
            // (d) owner's reverse CSR, bucket capacities (D34), selection
            if (nrecv > 0)
                c.launch("k_rec_count", [&] {
                    k_rec_count<<<static_cast<int>((nrecv + 255) / 256), 256, 0, stream>>>(rr, nrecv, R.S, nl, rpos.as<uint32_t>());
                });
            const int64_t rstride = static_cast<int64_t>(tf[0] > tf[1] ? tf[0] : tf[1]) + 1;
            const size_t bcap = 2 * (tf[0] + static_cast<size_t>(nl) * p) + tf[1] + static_cast<size_t>(nl) * p + 1;
            if (!rsrc.ensure(static_cast<size_t>(2 * rstride) * 4) || !bucket.ensure(bcap * 8)) {
                Z.set_err(KNNG_E_NOMEM, "device allocation failed");
                break;
            }
            R.S.rsrc = rsrc.as<uint32_t>();
            R.S.rstride = rstride;
            R.G.bucket = bucket.as<uint64_t>();
            const int64_t nb = scan_blocks(nl);
            c.launch("k_scan_reduce", [&] {
                k_scan_reduce<<<dim3(static_cast<unsigned>(nb), 3), kScanBlock, 0, stream>>>(R.S, nl, nb);
            });
            c.launch("k_scan_bsums", [&] { k_scan_bsums<<<3, kScanBlock, 0, stream>>>(R.S.bsum, nb); });
            c.launch("k_scan_final", [&] {
                k_scan_final<<<dim3(static_cast<unsigned>(nb), 3), kScanBlock, 0, stream>>>(R.S, nl, nb);
            });
            if (nrecv > 0)
                c.launch("k_rec_scatter", [&] {
                    k_rec_scatter<<<static_cast<int>((nrecv + 255) / 256), 256, 0, stream>>>(rr, nrecv, R.S, nl, rstride,
                                                                                          rpos.as<uint32_t>());
                });
            c.launch("k_rev_select", [&] {
                k_rev_select<<<R.warps_grid(nl, 8), 256, 8 * 64 * sizeof(uint32_t), stream>>>(R.D, R.S, tword, seed);
            });
            // (e) restricted join (D22) over the own nodes, record mode
            cudaMemsetAsync(nrec_d, 0, 8, stream);
            if (!R.join(t)) R.scatter(t);
            // (f) candidate records to the targets' owners, filed there
            cudaMemcpyAsync(hp + 4096, nrec_d, 8, cudaMemcpyDeviceToHost, stream);
            cudaMemsetAsync(dcnt, 0, static_cast<size_t>(gs) * 4, stream);
            if (!Z.sync()) break;
            const int64_t nrec = hp[4096];
            if (nrec > 0) {
                if (!rpos.ensure(static_cast<size_t>(nrec) * 4 + 4)) {
                    Z.set_err(KNNG_E_NOMEM, "device allocation failed");
                    break;
                }
                c.launch("k_cand_count", [&] {
                    k_cand_count<<<static_cast<int>((nrec + 255) / 256), 256, 0, stream>>>(R.G.rec_tgt, nrec_d, nl,
                                                                                        rpos.as<uint32_t>(), dcnt);
                });
            }
            Z.xchg(g0, g0 + gs, [&](int q) { return Xfer{q, dcnt + (q - g0), 4}; },
                   [&](int q) { return Xfer{q, rcvc + (q - g0), 4}; });
            cudaMemcpyAsync(rcvc + me, dcnt + me, 4, cudaMemcpyDeviceToDevice, stream);
            cudaMemcpyAsync(hc, dcnt, static_cast<size_t>(gs) * 4, cudaMemcpyDeviceToHost, stream);
            cudaMemcpyAsync(hc + gs, rcvc, static_cast<size_t>(gs) * 4, cudaMemcpyDeviceToHost, stream);
            if (!Z.sync()) break;
            std::vector<unsigned long long> cso(gs), cro(gs + 1);
            acc = 0;
            for (int j = 0; j < gs; ++j) {
                cso[j] = acc;
                acc += hc[j];
            }
            unsigned long long ra = 0;
            for (int j = 0; j < gs; ++j) {
                cro[j] = ra;
                ra += hc[gs + j];
            }
            cro[gs] = ra;
            const int64_t nin = static_cast<int64_t>(ra);
            cudaMemcpyAsync(binoff, cso.data(), cso.size() * 8, cudaMemcpyHostToDevice, stream);
            CandRec* co = candout.as<CandRec>();
            if (nrec > 0)
                c.launch("k_cand_scatter_owner", [&] {
                    k_cand_scatter_owner<<<static_cast<int>((nrec + 255) / 256), 256, 0, stream>>>(
                        R.G.rec_tgt, R.G.rec_key, nrec_d, nl, rpos.as<uint32_t>(), binoff, co);
                });
            if (!candin.ensure(static_cast<size_t>(nin) * 16 + 16)) {
                Z.set_err(KNNG_E_NOMEM, "device allocation failed");
                break;
            }
            CandRec* ci = candin.as<CandRec>();
            Z.xchg(g0, g0 + gs, [&](int q) { return Xfer{q, co + cso[q - g0], static_cast<size_t>(hc[q - g0]) * 16}; },
                   [&](int q) {
                       const int j = q - g0;
                       return Xfer{q, ci + cro[j], static_cast<size_t>(cro[j + 1] - cro[j]) * 16};
                   });
            cudaMemcpyAsync(ci + cro[me], co + cso[me], static_cast<size_t>(hc[me]) * 16, cudaMemcpyDeviceToDevice, stream);
            if (nin > 0)
                c.launch("k_cand_apply", [&] {
                    k_cand_apply<<<static_cast<int>((nin + 255) / 256), 256, 0, stream>>>(ci, nin, R.G);
                });
        }
        if (Z.failed()) break;
        // finalize (Alg. 3 line 11): merge the last buckets, then reserved
        if (mi > 0) R.merge_sample(1, 0, mi - 1);
        c.launch("k_ggm_finalize", [&] {
            k_ggm_finalize<<<grid, 256, 256 * sizeof(uint64_t), stream>>>(R.D, R.G, reserved);
        });
        cudaMemcpyAsync(cur.p, R.G.keys, static_cast<size_t>(tot) * 8, cudaMemcpyDeviceToDevice, stream);
        c.launch("k_keys_shift", [&] {
            k_keys_shift<<<static_cast<int>((tot + 255) / 256), 256, 0, stream>>>(cur.as<uint64_t>(), tot, G0);
        });
        R.collect_stats(mi);
        history.insert(history.end(), g_last_stats.begin(), g_last_stats.end());
    }
    if (Z.code != KNNG_OK) {
        c.finish();
        return fail(Z.code, "%s", Z.err.c_str());
    }
    // ---- 3. the own rows of the graph, global ids
    c.launch("k_export", [&] {
        k_export<<<static_cast<int>((nl * k + 255) / 256), 256, 0, stream>>>(cur.as<uint64_t>(), nl * k, out_ids, out_dists);
    });
    const knng_status s = c.finish();
    g_last_stats = history;
    return s;
}
