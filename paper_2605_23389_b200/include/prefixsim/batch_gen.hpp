// Prefix-aware batcher: Density First Search over the length index (PAPER
// Alg. 1).  API of the reference's batch_gen.hpp (BatchConstraints :13-24,
// Batch :26-41, refresh_batch_clocks :44-46, r_search :88-96, l_search :99-107,
// density_first_search :126-210).
//
// The member order of the returned Batch IS the GPU page-table order: the
// batch is admitted FIFO into SchedulerState::running (scheduler.hpp:216-226),
// whose order the executor turns into the CSR page table of the decode kernel.
//
// Semantics (reference code wins over the paper where they differ, SURVEY
// Appendix A 2-5):
//  * start at the oldest starving node of the scan depth, else the root;
//  * a leaf whose residents exceed b_max yields its greedy FIFO prefix;
//  * case 1 (blocks <= b_max, requests >= k_min): take the subtree;
//  * case 2 (blocks > b_max): descend to the child with most requests;
//  * case 3 (fits, too few): take the subtree, then expand through siblings
//    nearest-first (left siblings when the node has any, walking each
//    sibling's residents by descending leaf; else right siblings ascending),
//    stopping at the first request over the block budget or once k_min is met.
#pragma once

#include <prefixsim/kv_index.hpp>

#include <algorithm>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <vector>

namespace prefixsim {

struct BatchConstraints {
    std::int64_t b_max = 0;
    std::int64_t k_min = 36;
    double starvation_threshold_ms = 500.0;
    int starvation_scan_depth = 2;

    void validate() const {
        if (b_max < 1 || k_min < 1) throw std::invalid_argument("b_max and k_min must be >= 1");
    }
};

struct Batch {
    std::int64_t id = 0;
    std::vector<PoolResident> members;  // admission (= page-table) order
    std::int64_t total_blocks = 0;
    std::int64_t window_lo = 0, window_hi = 0;
    double created_ms = 0.0;
    bool starvation_override = false;
    std::vector<NodeRef> source_nodes;

    std::vector<RequestId> request_ids() const {
        std::vector<RequestId> ids(members.size());
        std::transform(members.begin(), members.end(), ids.begin(),
                       [](const PoolResident& m) { return m.id; });
        return ids;
    }
};

inline void refresh_batch_clocks(QuadTree& tree, const Batch& batch, double now_ms) {
    for (const NodeRef& n : batch.source_nodes) tree.touch_path(n, now_ms);
}

namespace dfs_detail {

// Greedy nearest-first admission over an ordered sibling list.  count_budget
// < 0 means unlimited.
inline std::vector<PoolResident> expand_siblings(const QuadTree& tree,
                                                 const std::vector<NodeRef>& siblings,
                                                 bool leaves_descending, std::int64_t block_budget,
                                                 std::int64_t count_budget) {
    std::vector<PoolResident> taken;
    std::int64_t spent = 0;
    for (const NodeRef& sib : siblings) {
        if (tree.request_count(sib) == 0) continue;
        std::vector<PoolResident> cand;
        const auto [first, last] = QuadTree::leaf_span(sib);
        if (leaves_descending) {
            // residents by descending leaf, FIFO inside a leaf (a stable sort of
            // the ascending collection by leaf, descending)
            for (std::int64_t leaf = last - 1; leaf >= first; --leaf) {
                tree.for_each_in_leaf(leaf, [&](const PoolResident& r) { cand.push_back(r); });
            }
        } else {
            cand = tree.collect_requests(sib);
        }
        for (const PoolResident& r : cand) {
            if (count_budget >= 0 && static_cast<std::int64_t>(taken.size()) >= count_budget) return taken;
            if (spent + r.kv_blocks > block_budget) return taken;
            spent += r.kv_blocks;
            taken.push_back(r);
        }
    }
    return taken;
}

inline std::vector<NodeRef> siblings_of(NodeRef node, bool leftward) {
    std::vector<NodeRef> order;
    const std::int64_t pos = node.index % 4;
    const std::int64_t base = node.index - pos;
    if (leftward) {
        for (std::int64_t k = pos - 1; k >= 0; --k) order.push_back({node.depth, base + k});
    } else {
        for (std::int64_t k = pos + 1; k < 4; ++k) order.push_back({node.depth, base + k});
    }
    return order;
}

}  // namespace dfs_detail

// Left siblings, nearest (rightmost) first, each walked from its highest leaf.
inline std::vector<PoolResident> r_search(const QuadTree& tree, NodeRef node, std::int64_t block_budget,
                                          std::int64_t count_budget = -1) {
    return dfs_detail::expand_siblings(tree, dfs_detail::siblings_of(node, true), true, block_budget,
                                       count_budget);
}

// Right siblings, nearest (leftmost) first, ascending leaves.
inline std::vector<PoolResident> l_search(const QuadTree& tree, NodeRef node, std::int64_t block_budget,
                                          std::int64_t count_budget = -1) {
    return dfs_detail::expand_siblings(tree, dfs_detail::siblings_of(node, false), false, block_budget,
                                       count_budget);
}

inline std::optional<Batch> density_first_search(QuadTree& tree, const BatchConstraints& constraints,
                                                 double now_ms, std::int64_t batch_id = 0,
                                                 bool update_clocks = true) {
    constraints.validate();
    if (tree.empty()) return std::nullopt;

    Batch out;
    out.id = batch_id;
    out.created_ms = now_ms;

    NodeRef at{0, 0};
    const std::vector<NodeRef> starving =
        tree.starving_nodes(constraints.starvation_scan_depth, now_ms, constraints.starvation_threshold_ms);
    if (!starving.empty()) {
        at = starving.front();
        out.starvation_override = true;
    }

    for (;;) {
        const std::int64_t blocks = tree.block_count(at);
        const std::int64_t count = tree.request_count(at);
        const bool fits = blocks <= constraints.b_max;

        if (!fits && at.depth == QuadTree::kLeafDepth) {  // overfull leaf: FIFO prefix
            std::int64_t spent = 0;
            bool full = false;
            tree.for_each_in_leaf(at.index, [&](const PoolResident& r) {
                if (full || spent + r.kv_blocks > constraints.b_max) {
                    full = true;
                    return;
                }
                spent += r.kv_blocks;
                out.members.push_back(r);
            });
            out.source_nodes.push_back(at);
            break;
        }
        if (fits && count >= constraints.k_min) {  // case 1
            out.members = tree.collect_requests(at);
            out.source_nodes.push_back(at);
            break;
        }
        if (!fits) {  // case 2
            at = tree.max_density_child(at);
            continue;
        }
        // case 3
        out.members = tree.collect_requests(at);
        out.source_nodes.push_back(at);
        if (at.depth > 0) {
            const std::int64_t block_budget = constraints.b_max - blocks;
            const std::int64_t count_budget = constraints.k_min - count;
            const std::vector<PoolResident> extra =
                (at.index % 4 > 0) ? r_search(tree, at, block_budget, count_budget)
                                   : l_search(tree, at, block_budget, count_budget);
            for (const PoolResident& r : extra) {
                out.members.push_back(r);
                out.source_nodes.push_back({QuadTree::kLeafDepth, QuadTree::leaf_of(r.prefix_len)});
            }
        }
        break;
    }

    if (out.members.empty()) return std::nullopt;
    out.window_lo = out.window_hi = out.members.front().prefix_len;
    for (const PoolResident& m : out.members) {
        out.total_blocks += m.kv_blocks;
        out.window_lo = std::min(out.window_lo, m.prefix_len);
        out.window_hi = std::max(out.window_hi, m.prefix_len);
    }
    if (update_clocks) refresh_batch_clocks(tree, out, now_ms);
    return out;
}

}  // namespace prefixsim
