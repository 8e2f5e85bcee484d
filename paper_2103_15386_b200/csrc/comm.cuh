// comm.cuh -- the exchange layer of the distributed GGM refine (SURVEY.md
// section 8(e) stage B).
//
// One operation: a grouped point-to-point exchange on a stream -- every rank
// posts the byte ranges it sends to each peer and the buffers it receives
// into, and the call returns once the transfers are ordered on the stream
// (NCCL semantics: stream-ordered, buffers reusable after the stream work).
// Two transports implement it:
//   * NcclComm -- one process per GPU, ncclSend/ncclRecv inside
//     ncclGroupStart/End over NVLink / NVSwitch.  libnccl is opened with
//     dlopen at knng_comm_init, so the library loads (and everything but the
//     sharded build runs) where NCCL is absent.
//   * LocalComm -- P ranks as P host threads of one process (one stream each,
//     any devices): a message is a device pointer + a CUDA event handed over
//     through a mailbox; the receiver copies with cudaMemcpyAsync after the
//     sender's event and hands a completion event back, which the sender's
//     stream waits on.  It exercises the whole distributed path on one GPU
//     (NCCL cannot put two ranks on one device), and single-process
//     multi-GPU use.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace knng {

struct Xfer {
    int peer;
    void* ptr;
    size_t bytes;
};

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // sends/recvs: at most one of each per peer; a rank's message to itself
    // is a plain device copy done by the caller.  Returns "" or an error.
    virtual std::string exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                                 cudaStream_t stream) = 0;
};

// ------------------------------------------------------------------ NCCL
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;

    static NcclApi& get() {
        static NcclApi api = [] {
            NcclApi a;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) {
                a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
                return a;
            }
            a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
            a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
            a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
            a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
            a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
            a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
            a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
            if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.Send || !a.Recv || !a.GroupStart ||
                !a.GroupEnd || !a.GetErrorString)
                a.error = "libnccl.so.2 lacks a required symbol";
            return a;
        }();
        return api;
    }
    bool ok() const { return error.empty(); }
};

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) NcclApi::get().CommDestroy(comm);
    }
    std::string exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                         cudaStream_t stream) override {
        NcclApi& A = NcclApi::get();
        ncclResult_t r = A.GroupStart();
        for (const Xfer& x : sends)
            if (r == ncclSuccess && x.bytes) r = A.Send(x.ptr, x.bytes, ncclUint8, x.peer, comm, stream);
        for (const Xfer& x : recvs)
            if (r == ncclSuccess && x.bytes) r = A.Recv(x.ptr, x.bytes, ncclUint8, x.peer, comm, stream);
        const ncclResult_t e = A.GroupEnd();
        if (r == ncclSuccess) r = e;
        return r == ncclSuccess ? std::string() : std::string("NCCL: ") + A.GetErrorString(r);
    }
};

// ------------------------------------------------------------------ local (threads)
struct Hub {
    struct Msg {
        const void* ptr;
        size_t bytes;
        cudaEvent_t ready;  // recorded on the sender's stream after its producers
    };
    int world;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<std::deque<Msg>> box;          // [src * world + dst]
    std::vector<std::deque<cudaEvent_t>> ack;  // [src * world + dst]: receiver's copy done
    explicit Hub(int w) : world(w), box(static_cast<size_t>(w) * w), ack(static_cast<size_t>(w) * w) {}
};

struct LocalComm final : Comm {
    std::shared_ptr<Hub> hub;
    std::string exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                         cudaStream_t stream) override {
        Hub& H = *hub;
        // 1. post every send (never blocks: no rank waits before posting)
        for (const Xfer& x : sends) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return "cudaEventCreate failed";
            cudaEventRecord(e, stream);
            std::lock_guard<std::mutex> lk(H.mu);
            H.box[static_cast<size_t>(rank) * H.world + x.peer].push_back({x.ptr, x.bytes, e});
            H.cv.notify_all();
        }
        // 2. receive: wait for the message, copy after the sender's event,
        //    hand back a completion event
        for (const Xfer& x : recvs) {
            Hub::Msg m;
            {
                std::unique_lock<std::mutex> lk(H.mu);
                auto& q = H.box[static_cast<size_t>(x.peer) * H.world + rank];
                H.cv.wait(lk, [&] { return !q.empty(); });
                m = q.front();
                q.pop_front();
            }
            if (m.bytes != x.bytes) return "local exchange: message size mismatch";
            cudaStreamWaitEvent(stream, m.ready, 0);
            cudaEventDestroy(m.ready);
            if (x.bytes) cudaMemcpyAsync(x.ptr, m.ptr, x.bytes, cudaMemcpyDefault, stream);
            cudaEvent_t done;
            if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess) return "cudaEventCreate failed";
            cudaEventRecord(done, stream);
            std::lock_guard<std::mutex> lk(H.mu);
            H.ack[static_cast<size_t>(x.peer) * H.world + rank].push_back(done);
            H.cv.notify_all();
        }
        // 3. the send buffers are reusable once the receivers' copies are done
        for (const Xfer& x : sends) {
            cudaEvent_t done;
            {
                std::unique_lock<std::mutex> lk(H.mu);
                auto& q = H.ack[static_cast<size_t>(rank) * H.world + x.peer];
                H.cv.wait(lk, [&] { return !q.empty(); });
                done = q.front();
                q.pop_front();
            }
            cudaStreamWaitEvent(stream, done, 0);
            cudaEventDestroy(done);
        }
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? std::string() : std::string("local exchange: ") + cudaGetErrorString(e);
    }
};

}  // namespace knng
