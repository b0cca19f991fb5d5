// Length-bucketing index of the host KV pool (the batcher's input).
//
// API of the reference's QuadTree (kv_index.hpp:31-247): a fixed fan-out-4
// tree over prefix lengths [1, 65536], 7 levels, 4096 leaves of 16 tokens
// (one leaf = one KV page of length), each node carrying (request count,
// block count, starvation clock); leaves hold residents in FIFO order and
// lengths beyond 65536 clamp into the last leaf.
//
// Implementation (B200 build): all 5461 nodes live in three flat arrays indexed
// by heap position (offset(d) = (4^d - 1) / 3), and each leaf's FIFO is an
// intrusive doubly-linked list over a slot arena, so remove() is O(depth)
// instead of a vector erase.  Observable behaviour (counters, clocks, FIFO
// order, exceptions) is the reference's.
#pragma once

#include <prefixsim/request.hpp>

#include <json.hpp>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace prefixsim {

struct PoolResident {
    RequestId id = 0;
    std::int64_t prefix_len = 0;
    std::int64_t kv_blocks = 0;
};

struct NodeRef {
    int depth = 0;
    std::int64_t index = 0;
    bool operator==(const NodeRef&) const = default;
};

class QuadTree {
 public:
    static constexpr int kLeafDepth = 6;
    static constexpr std::int64_t kRangeMax = 65536;
    static constexpr std::int64_t kLeafCount = 4096;
    static constexpr std::int64_t kLeafWidth = 16;

    QuadTree()
        : reqs_(kNodes, 0), blocks_(kNodes, 0), clock_(kNodes, 0.0), head_(kLeafCount, -1),
          tail_(kLeafCount, -1) {}

    static std::int64_t nodes_at(int depth) { return std::int64_t{1} << (2 * depth); }
    static std::int64_t clamp_len(std::int64_t prefix_len) { return std::min(prefix_len, kRangeMax); }
    static std::int64_t leaf_of(std::int64_t prefix_len) { return (clamp_len(prefix_len) - 1) >> 4; }

    static std::pair<std::int64_t, std::int64_t> node_range(NodeRef n) {
        const std::int64_t w = kRangeMax >> (2 * n.depth);
        const std::int64_t lo = n.index * w;
        return {lo + 1, lo + w};
    }
    static std::pair<std::int64_t, std::int64_t> leaf_span(NodeRef n) {
        const int sh = 2 * (kLeafDepth - n.depth);
        return {n.index << sh, (n.index + 1) << sh};
    }

    void insert(const PoolResident& r, double now_ms) {
        if (r.prefix_len < 1) throw std::invalid_argument("prefix_len must be >= 1");
        if (where_.find(r.id) != where_.end()) {
            throw std::invalid_argument("duplicate request id " + std::to_string(r.id));
        }
        const std::int64_t leaf = leaf_of(r.prefix_len);
        const int slot = alloc_slot(r, leaf);
        where_.emplace(r.id, slot);
        std::int64_t i = leaf;
        for (int d = kLeafDepth; d >= 0; --d, i >>= 2) {
            const std::size_t h = heap(d, i);
            if (reqs_[h] == 0 && clock_[h] < now_ms) clock_[h] = now_ms;  // waiting starts now
            reqs_[h] += 1;
            blocks_[h] += r.kv_blocks;
        }
        ++size_;
    }

    PoolResident remove(RequestId id) {
        const auto it = where_.find(id);
        if (it == where_.end()) {
            throw std::invalid_argument("request id not in tree: " + std::to_string(id));
        }
        const int slot = it->second;
        where_.erase(it);
        const PoolResident r = slots_[static_cast<std::size_t>(slot)].r;
        const std::int64_t leaf = slots_[static_cast<std::size_t>(slot)].leaf;
        unlink(slot);
        std::int64_t i = leaf;
        for (int d = kLeafDepth; d >= 0; --d, i >>= 2) {
            const std::size_t h = heap(d, i);
            reqs_[h] -= 1;
            blocks_[h] -= r.kv_blocks;
        }
        --size_;
        return r;
    }

    bool contains(RequestId id) const { return where_.find(id) != where_.end(); }
    std::int64_t size() const { return size_; }
    bool empty() const { return size_ == 0; }

    std::int64_t request_count(NodeRef n) const { return reqs_[heap(n.depth, n.index)]; }
    std::int64_t block_count(NodeRef n) const { return blocks_[heap(n.depth, n.index)]; }
    double last_batch_ms(NodeRef n) const { return clock_[heap(n.depth, n.index)]; }

    // Residents under n: leaves in ascending range order, FIFO inside a leaf.
    std::vector<PoolResident> collect_requests(NodeRef n) const {
        std::vector<PoolResident> out;
        out.reserve(static_cast<std::size_t>(request_count(n)));
        append_residents(n, out);
        return out;
    }

    template <typename F>
    void for_each_in_leaf(std::int64_t leaf, F&& f) const {
        for (int s = head_[static_cast<std::size_t>(leaf)]; s >= 0;
             s = slots_[static_cast<std::size_t>(s)].next) {
            f(slots_[static_cast<std::size_t>(s)].r);
        }
    }

    // Densest child by request count; first (lowest range) wins ties.
    NodeRef max_density_child(NodeRef n) const {
        if (n.depth >= kLeafDepth) throw std::invalid_argument("leaf has no children");
        NodeRef pick{-1, -1};
        std::int64_t most = 0;
        const std::int64_t first = n.index * 4;
        for (std::int64_t c = first; c < first + 4; ++c) {
            const std::int64_t cnt = reqs_[heap(n.depth + 1, c)];
            if (cnt > most) {
                most = cnt;
                pick = NodeRef{n.depth + 1, c};
            }
        }
        if (pick.depth < 0) throw std::invalid_argument("max_density_child of empty node");
        return pick;
    }

    // Raise the starvation clock of n and every ancestor to now (never lowers it).
    void touch_path(NodeRef n, double now_ms) {
        std::int64_t i = n.index;
        for (int d = n.depth; d >= 0; --d, i >>= 2) raise(heap(d, i), now_ms);
    }
    void touch_node(NodeRef n, double now_ms) { raise(heap(n.depth, n.index), now_ms); }

    // Non-empty nodes at scan_depth whose clock lags now by more than the
    // threshold, oldest clock first, index order on ties.
    std::vector<NodeRef> starving_nodes(int scan_depth, double now_ms, double threshold_ms) const {
        std::vector<NodeRef> found;
        const std::int64_t n = nodes_at(scan_depth);
        for (std::int64_t i = 0; i < n; ++i) {
            const std::size_t h = heap(scan_depth, i);
            if (reqs_[h] > 0 && now_ms - clock_[h] > threshold_ms) found.push_back({scan_depth, i});
        }
        std::sort(found.begin(), found.end(), [&](const NodeRef& a, const NodeRef& b) {
            const double ca = last_batch_ms(a), cb = last_batch_ms(b);
            return ca != cb ? ca < cb : a.index < b.index;
        });
        return found;
    }

    nlohmann::json dump_json() const { return render(NodeRef{0, 0}); }

 private:
    static constexpr std::size_t kNodes = 5461;  // (4^7 - 1) / 3

    struct Slot {
        PoolResident r;
        std::int64_t leaf = 0;
        int prev = -1, next = -1;
    };

    static std::size_t heap(int depth, std::int64_t index) {
        const std::int64_t base = ((std::int64_t{1} << (2 * depth)) - 1) / 3;
        return static_cast<std::size_t>(base + index);
    }

    void raise(std::size_t h, double now_ms) {
        if (clock_[h] < now_ms) clock_[h] = now_ms;
    }

    int alloc_slot(const PoolResident& r, std::int64_t leaf) {
        int s;
        if (!free_.empty()) {
            s = free_.back();
            free_.pop_back();
        } else {
            s = static_cast<int>(slots_.size());
            slots_.emplace_back();
        }
        Slot& sl = slots_[static_cast<std::size_t>(s)];
        sl.r = r;
        sl.leaf = leaf;
        sl.next = -1;
        sl.prev = tail_[static_cast<std::size_t>(leaf)];
        if (sl.prev >= 0) {
            slots_[static_cast<std::size_t>(sl.prev)].next = s;
        } else {
            head_[static_cast<std::size_t>(leaf)] = s;
        }
        tail_[static_cast<std::size_t>(leaf)] = s;
        return s;
    }

    void unlink(int s) {
        Slot& sl = slots_[static_cast<std::size_t>(s)];
        const auto leaf = static_cast<std::size_t>(sl.leaf);
        if (sl.prev >= 0) slots_[static_cast<std::size_t>(sl.prev)].next = sl.next;
        else head_[leaf] = sl.next;
        if (sl.next >= 0) slots_[static_cast<std::size_t>(sl.next)].prev = sl.prev;
        else tail_[leaf] = sl.prev;
        free_.push_back(s);
    }

    void append_residents(NodeRef n, std::vector<PoolResident>& out) const {
        if (reqs_[heap(n.depth, n.index)] == 0) return;
        if (n.depth == kLeafDepth) {
            for_each_in_leaf(n.index, [&](const PoolResident& r) { out.push_back(r); });
            return;
        }
        for (std::int64_t c = n.index * 4; c < n.index * 4 + 4; ++c) {
            append_residents(NodeRef{n.depth + 1, c}, out);
        }
    }

    nlohmann::json render(NodeRef n) const {
        nlohmann::json j;
        const auto [lo, hi] = node_range(n);
        j["range"] = {lo, hi};
        j["requests"] = request_count(n);
        j["blocks"] = block_count(n);
        j["last_batch_ms"] = last_batch_ms(n);
        if (n.depth == kLeafDepth) {
            nlohmann::json arr = nlohmann::json::array();
            for_each_in_leaf(n.index, [&](const PoolResident& r) {
                arr.push_back({{"id", r.id}, {"prefix_len", r.prefix_len}, {"blocks", r.kv_blocks}});
            });
            j["residents"] = std::move(arr);
        } else {
            nlohmann::json kids = nlohmann::json::array();
            for (std::int64_t c = n.index * 4; c < n.index * 4 + 4; ++c) {
                if (reqs_[heap(n.depth + 1, c)] > 0) kids.push_back(render(NodeRef{n.depth + 1, c}));
            }
            j["children"] = std::move(kids);
        }
        return j;
    }

    std::vector<std::int64_t> reqs_;
    std::vector<std::int64_t> blocks_;
    std::vector<double> clock_;
    std::vector<int> head_, tail_;
    std::vector<Slot> slots_;
    std::vector<int> free_;
    std::unordered_map<RequestId, int> where_;
    std::int64_t size_ = 0;
};

}  // namespace prefixsim
