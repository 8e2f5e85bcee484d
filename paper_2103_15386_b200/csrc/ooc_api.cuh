// ooc_api.cuh -- the paper's out-of-memory construction (D41),
// included at the end of knng_api.cu.
//
// "The large-scale dataset is partitioned into multiple shards.  Each shard
// is sufficiently small that is tractable by one GPU.  Thereafter, a k-NN
// graph for each shard is built by GNND and saved back to disk.  GGM is
// called to merge every two sub-graphs of two shards.  The merged graph is
// saved back to disk as two sub-graphs.  Each k-NN list in either sub-graphs
// retains the top-k neighbors of the corresponding object ... we can read and
// write the disk while merging graphs on GPU".
//
// Host memory plays the disk (the caller's buffers may be mmap'ed files):
//   phase 1: per shard g, vectors in (copy stream) -> knng_build (seed + g)
//            -> the sub-graph G_g back to host (pinned, local ids) and the
//            running lists R_g = G_g with global ids;
//   phase 2: for i < h (i outer): GGM(G_i, G_h) (knng_merge, Philox level
//            i S + h) -> M; k_ooc_fold: R(x) <- k smallest unique keys of
//            R(x) U M(x) for the rows of both shards.  Shard i (vectors, G_i,
//            R_i) stays resident for its whole row of pairs; shard h streams
//            through two device slots on the copy stream -- h+1's rows and
//            lists are read while (i, h) merges, R_h is written back after
//            its fold -- so the transfers hide behind the GPU work.
// Bit-identical to oracle.allpairs_build (same seeds, levels and folds; the
// fold is order-independent).
#pragma once

namespace knng {

// R(x) <- the k smallest unique keys of R(x) (global ids) U M(x) (merge-local
// ids: < nA -> baseA + id, else baseB + id - nA).  One warp per row; keys are
// canonical per (x, id) (D5), so a repeated id is a repeated key.
__global__ void k_ooc_fold(uint64_t* __restrict__ R, int64_t rows, int k, const uint32_t* __restrict__ m_ids,
                           const float* __restrict__ m_dists, int64_t nA, int64_t baseA, int64_t baseB) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const uint32_t lane = lane_id();
    extern __shared__ uint64_t fold_scratch[];  // 32 u64 per warp
    uint64_t* scr = fold_scratch + (threadIdx.x >> 5) * 32;
    const bool in = static_cast<int>(lane) < k;
    const uint64_t a = in ? R[r * k + lane] : kSentinel;
    uint64_t b = kSentinel;
    if (in) {
        const int64_t id = m_ids[r * k + lane];
        const int64_t g = id < nA ? baseA + id : baseB + (id - nA);
        b = make_key(m_dists[r * k + lane], static_cast<uint32_t>(g));
    }
    // drop M keys already in R (binary search in R's sorted copy), keep the
    // survivors' order (compaction by rank)
    __syncwarp();
    scr[lane] = a;
    __syncwarp();
    int pos = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
        if (scr[pos + step - 1] < b) pos += step;
    const bool keep = b != kSentinel && scr[pos] != b;
    const uint32_t km = __ballot_sync(kFull, keep);
    __syncwarp();
    scr[lane] = kSentinel;
    __syncwarp();
    if (keep) scr[__popc(km & lanemask_lt())] = b;
    __syncwarp();
    const uint64_t bs = scr[31 - lane];  // survivors, descending across lanes
    // the 32 smallest of two sorted lists form a bitonic sequence
    const uint64_t x = warp_bitonic_merge_u64(a < bs ? a : bs);
    if (in) R[r * k + lane] = x;
}

__global__ void k_ooc_keys(const uint32_t* __restrict__ ids, const float* __restrict__ dists, int64_t total,
                           uint32_t base, uint64_t* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < total) out[i] = make_key(dists[i], ids[i] + base);
}

}  // namespace knng

namespace {

bool is_host_accessible(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;  // unregistered pageable memory
    }
    return a.type != cudaMemoryTypeDevice;
}

}  // namespace

knng_status knng_build_ooc(const void* host_vectors, knng_dtype dt, int64_t n, int32_t d, int32_t k,
                           knng_metric metric, int32_t iters, int32_t merge_iters, int32_t sample_size, uint64_t seed,
                           int32_t shards, uint32_t* host_out_ids, float* host_out_dists, void* stream) {
    using namespace knng;
    knng_status s = check_common(dt, n, d, k, metric, sample_size);
    if (s) return s;
    if (k > 32) return fail(KNNG_E_USAGE, "GGM merges one-segment lists (k <= 32)");
    if (iters < 1 || iters > kMaxIters) return fail(KNNG_E_USAGE, "iters must be in [1, %d]", kMaxIters);
    if (merge_iters < 0 || merge_iters > kMaxIters) return fail(KNNG_E_USAGE, "merge_iters must be in [0, %d]", kMaxIters);
    if (shards < 1 || static_cast<int64_t>(shards) * shards > 0x7FFF)
        return fail(KNNG_E_USAGE, "shards must be in [1, 181] (merge levels i * S + h < 32768)");
    if (!host_vectors || !host_out_ids || !host_out_dists) return fail(KNNG_E_USAGE, "null pointer argument");
    if (!is_host_accessible(host_vectors) || !is_host_accessible(host_out_ids) || !is_host_accessible(host_out_dists))
        return fail(KNNG_E_USAGE, "knng_build_ooc takes host buffers");
    std::vector<int64_t> b(shards + 1);
    for (int g = 0; g <= shards; ++g) b[g] = static_cast<int64_t>(g) * n / shards;
    int64_t nmax = 0;
    for (int g = 0; g < shards; ++g) {
        const int64_t ng = b[g + 1] - b[g];
        if (ng <= k) return fail(KNNG_E_USAGE, "every shard needs more than k rows (n / shards = %lld)",
                                 static_cast<long long>(ng));
        nmax = std::max(nmax, ng);
    }
    const size_t esz = dt == KNNG_F32 ? 4 : 1;
    const size_t vrow = static_cast<size_t>(d) * esz, grow = static_cast<size_t>(k) * 4, krow = static_cast<size_t>(k) * 8;
    const size_t wsb = std::max(knng_build_workspace_bytes(dt, nmax, d, k, sample_size, metric),
                                shards > 1 ? knng_merge_workspace_bytes(dt, nmax, nmax, d, k, sample_size, metric) : 0);

    cudaStream_t cs = static_cast<cudaStream_t>(stream), ks = nullptr;
    // device: resident shard i (X, G ids/dists, R keys), two streamed slots
    // for h, the merge output, one workspace; host (pinned): the sub-graphs
    // G (local ids) and the running lists R (keys)
    struct Slot {
        char* X = nullptr;
        uint32_t* gi = nullptr;
        float* gd = nullptr;
        uint64_t* R = nullptr;
    } res, sl[2];
    char* dmem = nullptr;
    uint32_t* mi = nullptr;
    float* md = nullptr;
    uint32_t* ei = nullptr;  // final lists of one shard (ids / dists) on their way to the caller
    float* ed = nullptr;
    char* ws = nullptr;
    uint32_t* hG_ids = nullptr;
    float* hG_dists = nullptr;
    uint64_t* hR = nullptr;
    const size_t slotb = align_up(nmax * vrow) + 2 * align_up(nmax * grow) + align_up(nmax * krow);
    const size_t mb = 2 * align_up(2 * nmax * grow) + 2 * align_up(nmax * grow);  // merge output + export
    const size_t total = 3 * slotb + mb + align_up(wsb);
    cudaError_t e = cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dmem), total, cs);
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&hG_ids), static_cast<size_t>(n) * grow);
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&hG_dists), static_cast<size_t>(n) * grow);
    if (e == cudaSuccess && shards > 1) e = cudaMallocHost(reinterpret_cast<void**>(&hR), static_cast<size_t>(n) * krow);
    std::vector<cudaEvent_t> evs;
    auto ev = [&]() {
        cudaEvent_t x = nullptr;
        cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        evs.push_back(x);
        return x;
    };
    auto cleanup = [&](knng_status st) {
        cudaStreamSynchronize(cs);
        if (ks) cudaStreamSynchronize(ks);
        if (dmem) cudaFreeAsync(dmem, cs);
        cudaStreamSynchronize(cs);
        for (auto x : evs) cudaEventDestroy(x);
        if (ks) cudaStreamDestroy(ks);
        if (hG_ids) cudaFreeHost(hG_ids);
        if (hG_dists) cudaFreeHost(hG_dists);
        if (hR) cudaFreeHost(hR);
        return st;
    };
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cleanup(fail(e == cudaErrorMemoryAllocation ? KNNG_E_NOMEM : KNNG_E_CUDA, "knng_build_ooc: %s",
                            cudaGetErrorString(e)));
    }
    {
        char* p = dmem;
        for (Slot* t : {&res, &sl[0], &sl[1]}) {
            t->X = p;
            p += align_up(nmax * vrow);
            t->gi = reinterpret_cast<uint32_t*>(p);
            p += align_up(nmax * grow);
            t->gd = reinterpret_cast<float*>(p);
            p += align_up(nmax * grow);
            t->R = reinterpret_cast<uint64_t*>(p);
            p += align_up(nmax * krow);
        }
        mi = reinterpret_cast<uint32_t*>(p);
        p += align_up(2 * nmax * grow);
        md = reinterpret_cast<float*>(p);
        p += align_up(2 * nmax * grow);
        ei = reinterpret_cast<uint32_t*>(p);
        p += align_up(nmax * grow);
        ed = reinterpret_cast<float*>(p);
        p += align_up(nmax * grow);
        ws = p;
    }
    const char* hX = static_cast<const char*>(host_vectors);
    auto nrows = [&](int g) { return b[g + 1] - b[g]; };
    std::vector<knng_iter_stats> hist;
    auto put_stats = [&]() { hist.insert(hist.end(), g_last_stats.begin(), g_last_stats.end()); };
    auto check = [&](const char* where) -> knng_status {
        const cudaError_t x = cudaGetLastError();
        if (x != cudaSuccess) return fail(KNNG_E_CUDA, "knng_build_ooc (%s): %s", where, cudaGetErrorString(x));
        return KNNG_OK;
    };

    // ---- phase 1: sub-graph of every shard; the next shard's rows are
    // copied in while this one builds
    cudaEvent_t in_done[2] = {ev(), ev()}, slot_free[2] = {ev(), ev()};
    auto load_x = [&](int g, int slot) {
        cudaStreamWaitEvent(ks, slot_free[slot], 0);
        cudaMemcpyAsync(sl[slot].X, hX + static_cast<size_t>(b[g]) * vrow, nrows(g) * vrow, cudaMemcpyHostToDevice, ks);
        cudaEventRecord(in_done[slot], ks);
    };
    cudaEventRecord(slot_free[0], cs);
    cudaEventRecord(slot_free[1], cs);
    load_x(0, 0);
    for (int g = 0; g < shards; ++g) {
        const int slot = g & 1;
        if (g + 1 < shards) load_x(g + 1, slot ^ 1);
        cudaStreamWaitEvent(cs, in_done[slot], 0);
        s = knng_build(sl[slot].X, dt, nrows(g), d, k, metric, iters, sample_size, seed + g, sl[slot].gi, sl[slot].gd,
                       ws, wsb, cs);
        if (s) return cleanup(s);
        put_stats();
        if (shards == 1) {
            cudaMemcpyAsync(host_out_ids, sl[slot].gi, nrows(g) * grow, cudaMemcpyDeviceToHost, cs);
            cudaMemcpyAsync(host_out_dists, sl[slot].gd, nrows(g) * grow, cudaMemcpyDeviceToHost, cs);
            break;
        }
        // G_g to host (the merges' input) and R_g = G_g with global ids
        knng::k_ooc_keys<<<static_cast<unsigned>((nrows(g) * k + 255) / 256), 256, 0, cs>>>(
            sl[slot].gi, sl[slot].gd, nrows(g) * k, static_cast<uint32_t>(b[g]), sl[slot].R);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        cudaEvent_t built = ev();
        cudaEventRecord(built, cs);
        cudaStreamWaitEvent(ks, built, 0);
        cudaMemcpyAsync(hG_ids + static_cast<size_t>(b[g]) * k, sl[slot].gi, nrows(g) * grow, cudaMemcpyDeviceToHost, ks);
        cudaMemcpyAsync(hG_dists + static_cast<size_t>(b[g]) * k, sl[slot].gd, nrows(g) * grow, cudaMemcpyDeviceToHost, ks);
        cudaMemcpyAsync(hR + static_cast<size_t>(b[g]) * k, sl[slot].R, nrows(g) * krow, cudaMemcpyDeviceToHost, ks);
        cudaEventRecord(slot_free[slot], ks);  // the slot may be refilled after its copies out
        if ((s = check("build"))) return cleanup(s);
    }
    if (shards > 1) {
        // ---- phase 2: every pair once, i outer; shard h streams through
        // the two slots
        auto load_shard = [&](int g, Slot& t, cudaEvent_t wait_free, cudaEvent_t done) {
            cudaStreamWaitEvent(ks, wait_free, 0);
            cudaMemcpyAsync(t.X, hX + static_cast<size_t>(b[g]) * vrow, nrows(g) * vrow, cudaMemcpyHostToDevice, ks);
            cudaMemcpyAsync(t.gi, hG_ids + static_cast<size_t>(b[g]) * k, nrows(g) * grow, cudaMemcpyHostToDevice, ks);
            cudaMemcpyAsync(t.gd, hG_dists + static_cast<size_t>(b[g]) * k, nrows(g) * grow, cudaMemcpyHostToDevice, ks);
            cudaMemcpyAsync(t.R, hR + static_cast<size_t>(b[g]) * k, nrows(g) * krow, cudaMemcpyHostToDevice, ks);
            cudaEventRecord(done, ks);
        };
        cudaEvent_t res_free = ev(), res_in = ev();
        cudaEventRecord(res_free, ks);  // phase 1's copies out precede every reload
        cudaEventRecord(slot_free[0], ks);
        cudaEventRecord(slot_free[1], ks);
        const int fold_wpb = 8;
        cudaEvent_t exp_free = ev();
        cudaEventRecord(exp_free, ks);
        // a finished shard's lists leave as ids / dists, straight into the
        // caller's buffers
        auto export_final = [&](int g, const uint64_t* Rd) {
            cudaStreamWaitEvent(cs, exp_free, 0);
            k_export<<<static_cast<unsigned>((nrows(g) * k + 255) / 256), 256, 0, cs>>>(Rd, nrows(g) * k, ei, ed);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            cudaEvent_t x = ev();
            cudaEventRecord(x, cs);
            cudaStreamWaitEvent(ks, x, 0);
            cudaMemcpyAsync(host_out_ids + static_cast<size_t>(b[g]) * k, ei, nrows(g) * grow, cudaMemcpyDeviceToHost, ks);
            cudaMemcpyAsync(host_out_dists + static_cast<size_t>(b[g]) * k, ed, nrows(g) * grow, cudaMemcpyDeviceToHost, ks);
            cudaEventRecord(exp_free, ks);
        };
        for (int i = 0; i + 1 < shards; ++i) {
            load_shard(i, res, res_free, res_in);
            cudaStreamWaitEvent(cs, res_in, 0);
            int slot = 0, last_slot = 0;
            load_shard(i + 1, sl[slot], slot_free[slot], in_done[slot]);
            for (int h = i + 1; h < shards; ++h, slot ^= 1) {
                if (h + 1 < shards) load_shard(h + 1, sl[slot ^ 1], slot_free[slot ^ 1], in_done[slot ^ 1]);
                cudaStreamWaitEvent(cs, in_done[slot], 0);
                const int64_t nA = nrows(i), nB = nrows(h);
                s = knng_merge(res.X, nA, res.gi, res.gd, sl[slot].X, nB, sl[slot].gi, sl[slot].gd, dt, d, k, metric,
                               merge_iters, sample_size, i * shards + h, seed, mi, md, ws, wsb, cs);
                if (s) return cleanup(s);
                put_stats();
                const size_t fsm = fold_wpb * 32 * sizeof(uint64_t);
                knng::k_ooc_fold<<<static_cast<unsigned>((nA + fold_wpb - 1) / fold_wpb), fold_wpb * 32, fsm, cs>>>(
                    res.R, nA, k, mi, md, nA, b[i], b[h]);
                knng::k_ooc_fold<<<static_cast<unsigned>((nB + fold_wpb - 1) / fold_wpb), fold_wpb * 32, fsm, cs>>>(
                    sl[slot].R, nB, k, mi + nA * k, md + nA * k, nA, b[i], b[h]);
                g_launches.fetch_add(2, std::memory_order_relaxed);
                // R_h back to host, then the slot may be refilled
                cudaEvent_t folded = ev();
                cudaEventRecord(folded, cs);
                cudaStreamWaitEvent(ks, folded, 0);
                cudaMemcpyAsync(hR + static_cast<size_t>(b[h]) * k, sl[slot].R, nB * krow, cudaMemcpyDeviceToHost, ks);
                cudaEventRecord(slot_free[slot], ks);
                last_slot = slot;
                if ((s = check("merge"))) return cleanup(s);
            }
            // R_i is final after its row of pairs (and the last shard's
            // after the last pair)
            export_final(i, res.R);
            if (i + 2 == shards) export_final(i + 1, sl[last_slot].R);
            cudaEvent_t done_i = ev();
            cudaEventRecord(done_i, cs);
            cudaStreamWaitEvent(ks, done_i, 0);
            cudaEventRecord(res_free, ks);
            if ((s = check("export"))) return cleanup(s);
        }
    }
    e = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ks);
    if (e != cudaSuccess) return cleanup(fail(KNNG_E_CUDA, "knng_build_ooc: %s", cudaGetErrorString(e)));
    knng_status out = cleanup(KNNG_OK);
    g_last_stats = hist;
    return out;
}
