// host_staging.hpp — host↔device copies for pageable user memory.
//
// The drop-in API receives points in a std::vector (lsqfit::Dataset,
// reference dataset.hpp:36): pageable memory, which the CUDA driver copies
// through its own small staging buffers at ~11 GB/s on the B200 box (vs
// ~55 GB/s from pinned memory, profiles/r01_h2d.json). Here pageable
// transfers go through two pinned staging buffers filled / drained by a small
// persistent thread pool: the CPU copy of piece i+1 overlaps the DMA of piece
// i. Pinned (page-locked / registered) pointers and small copies go straight
// to cudaMemcpyAsync.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace lsq_host {

// Persistent worker pool running one parallel memcpy at a time.
class CopyPool {
public:
    explicit CopyPool(int threads) {
        parts_ = threads;
        try {
            for (int i = 0; i < threads - 1; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
        } catch (...) {
            shutdown();  // join the workers already started, then report
            throw;
        }
    }
    ~CopyPool() { shutdown(); }
    CopyPool(const CopyPool&) = delete;
    CopyPool& operator=(const CopyPool&) = delete;

    // memcpy split over `parts_` threads (the caller takes slice 0).
    void copy(void* dst, const void* src, size_t bytes) {
        if (parts_ <= 1 || bytes < (size_t(4) << 20)) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<unsigned char*>(dst);
            src_ = static_cast<const unsigned char*>(src);
            bytes_ = bytes;
            pending_ = parts_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        slice(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

private:
    void shutdown() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_)
            if (t.joinable()) t.join();
        workers_.clear();
    }

    void slice(int i) {
        const size_t per = (bytes_ / parts_ + 63) & ~size_t(63);
        const size_t lo = std::min(bytes_, per * size_t(i));
        const size_t hi = std::min(bytes_, lo + per);
        if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void loop(int i) {
        unsigned long seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            if (stop_) return;
            lk.unlock();
            slice(i);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    unsigned char* dst_ = nullptr;
    const unsigned char* src_ = nullptr;
    size_t bytes_ = 0;
    int parts_ = 1;
    int pending_ = 0;
    unsigned long gen_ = 0;
    bool stop_ = false;
};

inline bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Two pinned staging buffers + events marking when each is free again.
class Stager {
public:
    static constexpr size_t kPiece = size_t(64) << 20;  // bytes per staged piece

    ~Stager() { release(); }

    cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
        if (bytes < (size_t(8) << 20) || is_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        cudaError_t e = ensure();
        if (e != cudaSuccess) return e;
        size_t i = 0;
        for (size_t off = 0; off < bytes; off += kPiece, ++i) {
            const int b = int(i & 1);
            const size_t len = std::min(kPiece, bytes - off);
            if ((e = cudaEventSynchronize(free_[b])) != cudaSuccess) return e;  // previous DMA out of buf b done
            pool_->copy(buf_[b], static_cast<const unsigned char*>(src) + off, len);
            if ((e = cudaMemcpyAsync(static_cast<unsigned char*>(dst) + off, buf_[b], len, cudaMemcpyHostToDevice, st)) !=
                cudaSuccess)
                return e;
            if ((e = cudaEventRecord(free_[b], st)) != cudaSuccess) return e;
        }
        return cudaSuccess;
    }

    // Synchronous from the host's point of view for pageable destinations.
    cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
        if (bytes < (size_t(8) << 20) || is_pinned(dst)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
        cudaError_t e = ensure();
        if (e != cudaSuccess) return e;
        const size_t np = (bytes + kPiece - 1) / kPiece;
        size_t prev_off = 0, prev_len = 0;
        for (size_t i = 0; i <= np; ++i) {  // piece i in flight while piece i-1 drains
            const int b = int(i & 1);
            const size_t off = i * kPiece;
            const size_t len = i < np ? std::min(kPiece, bytes - off) : 0;
            if (len) {
                if ((e = cudaEventSynchronize(free_[b])) != cudaSuccess) return e;
                if ((e = cudaMemcpyAsync(buf_[b], static_cast<const unsigned char*>(src) + off, len,
                                         cudaMemcpyDeviceToHost, st)) != cudaSuccess)
                    return e;
                if ((e = cudaEventRecord(full_[b], st)) != cudaSuccess) return e;
            }
            if (i > 0) {  // drain the previous piece while this one is in flight
                const int pb = b ^ 1;
                if ((e = cudaEventSynchronize(full_[pb])) != cudaSuccess) return e;
                pool_->copy(static_cast<unsigned char*>(dst) + prev_off, buf_[pb], prev_len);
                if ((e = cudaEventRecord(free_[pb], st)) != cudaSuccess) return e;
            }
            prev_off = off;
            prev_len = len;
            if (!len) break;
        }
        return cudaSuccess;
    }

    void release() {
        for (int b = 0; b < 2; ++b) {
            if (buf_[b]) cudaFreeHost(buf_[b]);
            if (free_[b]) cudaEventDestroy(free_[b]);
            if (full_[b]) cudaEventDestroy(full_[b]);
            buf_[b] = nullptr;
            free_[b] = full_[b] = nullptr;
        }
        delete pool_;
        pool_ = nullptr;
    }

private:
    cudaError_t ensure() {
        if (pool_) return cudaSuccess;
        for (int b = 0; b < 2; ++b) {  // idempotent: a failed first attempt can be retried
            cudaError_t e;
            if (!buf_[b] && (e = cudaMallocHost(&buf_[b], kPiece)) != cudaSuccess) return e;
            if (!free_[b] && (e = cudaEventCreateWithFlags(&free_[b], cudaEventDisableTiming)) != cudaSuccess) return e;
            if (!full_[b] && (e = cudaEventCreateWithFlags(&full_[b], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        const char* env = std::getenv("LSQFIT_CUDA_HOST_THREADS");
        int threads = env ? std::atoi(env) : int(std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2)));
        try {  // no exception may cross the C ABI
            pool_ = new CopyPool(std::max(1, threads));
        } catch (...) {
            pool_ = nullptr;
            return cudaErrorMemoryAllocation;
        }
        return cudaSuccess;
    }

    void* buf_[2] = {nullptr, nullptr};
    cudaEvent_t free_[2] = {nullptr, nullptr};
    cudaEvent_t full_[2] = {nullptr, nullptr};
    CopyPool* pool_ = nullptr;
};

}  // namespace lsq_host
