// Relocation planner: cost-model placement of prefix groups on
// workers, the beam search of PAPER.md Alg. 1 (§3.2 "Beam Search with Incremental Cost",
// PAPER.md:188-236) scored with the cost functions of §3.2 "Cost Functions"
// (PAPER.md:315-332).  Host-only; the moves it returns are executed with the migration
// path (halo_migrate_send/recv, halo_prefix_clone, halo_prefix_fetch), which is how "KV
// blocks move between GPUs when the cost model relocates a DAG node" (north_star).
//
// Per iteration (Alg. 1 lines 3-12):
//   V_r      = the ops_per_iter unassigned items of largest e_v (the paper's top-|D| ready
//              operators; prefix groups have no dependencies, so all unassigned are ready);
//   Assign   = every combination of one option per item of V_r, an option being a single
//              worker or (conditions (i), (ii) of PAPER.md:236) a replica set;
//   Cost(f') = C_a(f') + C_r(f');
//   B        = Top(B', w) by (cost, lexicographic assignment).
// The readings of e_v, p_v, gamma/sigma/lambda are listed in include/halo_attn.h and
// DESIGN.md §5.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <numeric>
#include <vector>

#include "runtime.h"

namespace {

struct State {
    std::vector<uint64_t> mask;  // per item (0 = unassigned)
    std::vector<double> load;    // C_a^d
    double cost = 0.0;           // C_a + C_r
};

bool state_less(const State &a, const State &b) {
    if (a.cost != b.cost) return a.cost < b.cost;
    return a.mask < b.mask;  // lexicographic in item order
}

halo_status bad(const char *msg) { return halo::report_error(HALO_EINVAL, msg); }

// p_v(d): context preparation of item v on worker d ("context preparation
// latency"; here the KV relocation of §3.3).
double prep_cost(const halo_place_item &it, int d, double link) {
    if (it.home == d) return 0.0;
    if (it.home >= 0) return it.kv_bytes / link;
    return it.prep_s;
}

// The options of item v in state s: single workers, then replica sets of k = 2..kmax.
void options_for(const halo_place_item &it, int workers, bool replicate, const State &s,
                 std::vector<uint64_t> &out) {
    out.clear();
    for (int d = 0; d < workers; ++d) out.push_back(1ull << d);
    if (!replicate) return;
    const int kmax = std::min(it.max_replicas, workers);
    // home first, then the least-loaded other workers (ties: lower index)
    std::vector<int> order(workers);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const bool ha = a == it.home, hb = b == it.home;
        if (ha != hb) return ha;
        return s.load[a] < s.load[b];
    });
    uint64_t m = 1ull << order[0];
    for (int k = 2; k <= kmax; ++k) {
        m |= 1ull << order[k - 1];
        out.push_back(m);
    }
}

}  // namespace

extern "C" halo_status halo_place_groups(const halo_place_config *cfg, int32_t n, const halo_place_item *items,
                                         uint64_t *worker_mask, double *load, double *cost,
                                         halo_place_move *moves, int32_t move_cap, int32_t *n_moves) {
    try {
        if (cfg == nullptr || items == nullptr || worker_mask == nullptr || cost == nullptr || n_moves == nullptr)
            return bad("halo_place_groups: null argument");
        const int D = cfg->workers;
        if (n < 1) return bad("halo_place_groups: n must be >= 1");
        if (D < 1 || D > 64) return bad("halo_place_groups: workers must be in [1, 64]");
        if (cfg->beam_width < 1) return bad("halo_place_groups: beam_width must be >= 1");
        if (cfg->ops_per_iter < 1 || cfg->ops_per_iter > D) return bad("halo_place_groups: ops_per_iter must be in [1, workers]");
        if (!(cfg->beta >= 0.0) || !std::isfinite(cfg->beta)) return bad("halo_place_groups: beta must be finite and >= 0");
        if (!(cfg->link_bytes_per_s > 0.0)) return bad("halo_place_groups: link_bytes_per_s must be > 0");
        if (moves == nullptr && move_cap != 0) return bad("halo_place_groups: moves is NULL but move_cap != 0");
        double total = 0.0;
        for (int i = 0; i < n; ++i) {
            const halo_place_item &it = items[i];
            if (!(it.exec_s >= 0.0) || !std::isfinite(it.exec_s) || !(it.kv_bytes >= 0.0) ||
                !std::isfinite(it.kv_bytes) || !(it.prep_s >= 0.0) || !std::isfinite(it.prep_s))
                return bad("halo_place_groups: exec_s, kv_bytes, prep_s must be finite and >= 0");
            if (it.home < -1 || it.home >= D) return bad("halo_place_groups: home must be -1 or a worker index");
            if (it.max_replicas < 1) return bad("halo_place_groups: max_replicas must be >= 1");
            total += it.exec_s;
        }
        const double link = cfg->link_bytes_per_s;
        const double mbeta = std::pow((double)D, cfg->beta);

        // V_r order: decreasing e_v, ties lower index
        std::vector<int> rank(n);
        std::iota(rank.begin(), rank.end(), 0);
        std::stable_sort(rank.begin(), rank.end(), [&](int a, int b) { return items[a].exec_s > items[b].exec_s; });

        std::vector<State> beam(1);
        beam[0].mask.assign(n, 0);
        beam[0].load.assign(D, 0.0);
        beam[0].cost = total / mbeta;  // C_a(empty) = 0, C_r = all work
        double remaining = total;
        int next = 0;
        std::vector<State> cand;
        std::vector<std::vector<uint64_t>> opts;
        while (next < n) {
            const int nv = std::min(cfg->ops_per_iter, n - next);
            const int unassigned = n - next;
            double rem_after = remaining;
            for (int j = 0; j < nv; ++j) rem_after -= items[rank[next + j]].exec_s;
            if (rem_after < 0.0) rem_after = 0.0;
            cand.clear();
            for (const State &s : beam) {
                // options per item of V_r, in this state (replica sets depend on its loads)
                opts.assign(nv, {});
                double combos = 1.0;
                for (int j = 0; j < nv; ++j) {
                    const halo_place_item &it = items[rank[next + j]];
                    const bool replicate = it.max_replicas > 1 && unassigned < D && it.exec_s * D >= total;
                    options_for(it, D, replicate, s, opts[j]);
                    combos *= (double)opts[j].size();
                }
                if (combos * (double)beam.size() > (double)(1 << 20))
                    return bad("halo_place_groups: more than 2^20 candidates in one iteration "
                               "(lower ops_per_iter or beam_width)");
                std::vector<int> pick(nv, 0);
                for (;;) {
                    State c;
                    c.mask = s.mask;
                    c.load = s.load;
                    for (int j = 0; j < nv; ++j) {
                        const int v = rank[next + j];
                        const halo_place_item &it = items[v];
                        const uint64_t m = opts[j][pick[j]];
                        const int k = __builtin_popcountll(m);
                        const double share = it.exec_s / std::pow((double)k, cfg->beta);
                        c.mask[v] = m;
                        for (int d = 0; d < D; ++d)
                            if (m >> d & 1ull) c.load[d] += share + prep_cost(it, d, link);
                    }
                    c.cost = *std::max_element(c.load.begin(), c.load.end()) + rem_after / mbeta;
                    cand.push_back(std::move(c));
                    int j = nv - 1;  // mixed-radix increment, last item fastest
                    while (j >= 0 && ++pick[j] == (int)opts[j].size()) pick[j--] = 0;
                    if (j < 0) break;
                }
            }
            const size_t keep = std::min(cand.size(), (size_t)cfg->beam_width);
            std::partial_sort(cand.begin(), cand.begin() + keep, cand.end(), state_less);
            cand.resize(keep);
            beam.swap(cand);
            remaining = rem_after;
            next += nv;
        }
        const State &best = beam[0];  // sorted: lowest (cost, assignment)
        for (int i = 0; i < n; ++i) worker_mask[i] = best.mask[i];
        if (load != nullptr)
            for (int d = 0; d < D; ++d) load[d] = best.load[d];
        *cost = best.cost;

        // the moves that realise the placement
        int32_t nm = 0;
        for (int i = 0; i < n; ++i) {
            const halo_place_item &it = items[i];
            const uint64_t m = best.mask[i];
            int last = -1;
            for (int d = 0; d < D; ++d)
                if ((m >> d & 1ull) && d != it.home) last = d;
            for (int d = 0; d < D; ++d) {
                if (!(m >> d & 1ull) || d == it.home) continue;
                if (nm < move_cap) {
                    halo_place_move &mv = moves[nm];
                    mv.item = i;
                    mv.src = it.home;
                    mv.dst = d;
                    const bool home_kept = it.home >= 0 && (m >> it.home & 1ull);
                    mv.mode = (it.home >= 0 && !home_kept && d == last) ? 0 : 1;
                    mv.seconds = prep_cost(it, d, link);
                }
                ++nm;
            }
        }
        *n_moves = nm;
        if (nm > move_cap) {
            char buf[128];
            snprintf(buf, sizeof buf, "halo_place_groups: %d moves, move_cap %d", nm, move_cap);
            return halo::report_error(HALO_ENOMEM, buf);
        }
        return HALO_OK;
    } catch (const std::bad_alloc &) {
        return halo::report_error(HALO_ENOMEM, "halo_place_groups: host allocation failed");
    } catch (...) {
        return halo::report_error(HALO_EINVAL, "halo_place_groups: internal error");
    }
}
