// First-fit sub-allocator over the caller-bound device workspace (host-side
// bookkeeping only; all returned pointers are device pointers).  Work is
// stream-ordered on one stream, so a freed block may be reused by later work
// on the same stream without synchronisation.
#pragma once
#include <cstddef>
#include <cstdint>
#include <map>

#include "dot_common.cuh"

namespace dot {

class Arena {
public:
    static constexpr size_t kAlign = 256;

    void reset(void* base, size_t bytes) {
        base_ = static_cast<char*>(base);
        size_ = bytes;
        free_.clear();
        used_.clear();
        if (bytes) free_[0] = bytes;
    }
    bool bound() const { return base_ != nullptr; }

    void* alloc(size_t bytes) {
        bytes = (bytes + kAlign - 1) / kAlign * kAlign;
        if (bytes == 0) bytes = kAlign;
        for (auto it = free_.begin(); it != free_.end(); ++it) {
            if (it->second >= bytes) {
                size_t off = it->first, len = it->second;
                free_.erase(it);
                if (len > bytes) free_[off + bytes] = len - bytes;
                used_[off] = bytes;
                return base_ + off;
            }
        }
        throw Error(DOT_ERR_WORKSPACE, "workspace exhausted: need " + std::to_string(bytes) +
                                           " bytes, largest free block " + std::to_string(largest_free()));
    }

    void release(void* p) {
        if (!p) return;
        size_t off = static_cast<char*>(p) - base_;
        auto it = used_.find(off);
        if (it == used_.end()) return;
        size_t len = it->second;
        used_.erase(it);
        auto nx = free_.lower_bound(off);
        if (nx != free_.end() && off + len == nx->first) {   // merge with next
            len += nx->second;
            nx = free_.erase(nx);
        }
        if (nx != free_.begin()) {                           // merge with previous
            auto pv = std::prev(nx);
            if (pv->first + pv->second == off) {
                pv->second += len;
                return;
            }
        }
        free_[off] = len;
    }

    size_t capacity() const { return size_; }
    size_t used_bytes() const {
        size_t u = 0;
        for (const auto& kv : used_) u += kv.second;
        return u;
    }
    size_t largest_free() const {
        size_t m = 0;
        for (auto& kv : free_) m = kv.second > m ? kv.second : m;
        return m;
    }

private:
    char* base_ = nullptr;
    size_t size_ = 0;
    std::map<size_t, size_t> free_, used_;
};

// RAII device block from an Arena.
template <class T>
class DBuf {
public:
    DBuf() = default;
    DBuf(Arena& a, size_t count) : a_(&a), p_(static_cast<T*>(a.alloc(count * sizeof(T)))), n_(count) {}
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : a_(o.a_), p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            a_ = o.a_;
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
        }
        return *this;
    }
    ~DBuf() { reset(); }
    void reset() {
        if (p_ && a_) a_->release(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    explicit operator bool() const { return p_ != nullptr; }

private:
    Arena* a_ = nullptr;
    T* p_ = nullptr;
    size_t n_ = 0;
};

}  // namespace dot
