// Pass planner; see plan.h for the model.
#include "plan.h"

#include <algorithm>
#include <stdexcept>

namespace svgb {

static inline int popc(uint64_t v) { return __builtin_popcountll(v); }
static inline uint64_t low_mask(int b) { return b >= 64 ? ~0ull : ((1ull << b) - 1); }

GateShape gate_shape(const svg_gate& g) {
  GateShape s;
  uint64_t tmask = 0;
  for (int j = 0; j < g.ntargets; ++j) tmask |= 1ull << g.targets[j];
  s.flip = (g.form == SVG_FORM_PAULI) ? g.x_mask : tmask;
  s.touch = tmask | g.ctrl_mask;
  s.nderiv = g.nderiv;
  return s;
}

// Fill the tile set up to k qubits with the lowest unused qubits.
static uint64_t pad_tile(uint64_t q, int n, int k) {
  for (int i = 0; i < n && popc(q) < k; ++i) q |= 1ull << i;
  return q;
}

Pass plan_one_pass(const std::vector<GateShape>& shapes, std::vector<char>& done, const PlanParams& pp,
                   uint64_t forbidden_flip, uint64_t allowed_flip) {
  const int G = static_cast<int>(shapes.size());
  // every qubit counts for the early exit, including global (rank) positions
  uint64_t all = 0;
  for (const GateShape& s : shapes) all |= s.touch;
  Pass p;
  uint64_t q = low_mask(pp.b);
  uint64_t flip_blocked = 0, diag_blocked = 0;
  int derivs = 0;
  for (int i = 0; i < G; ++i) {
    if (done[i]) continue;
    const GateShape& s = shapes[i];
    const uint64_t diag = s.touch & ~s.flip;
    bool ok = !(s.touch & flip_blocked) && !(s.flip & diag_blocked) && !(s.flip & forbidden_flip) &&
              !(s.flip & ~allowed_flip);
    ok = ok && popc(q | s.flip) <= pp.k;
    ok = ok && static_cast<int>(p.items.size()) < pp.max_items;
    ok = ok && derivs + s.nderiv <= pp.max_derivs;
    if (ok) {
      q |= s.flip;
      p.items.push_back(i);
      derivs += s.nderiv;
      done[i] = 1;
    } else {
      flip_blocked |= s.flip;
      diag_blocked |= diag;
      if ((flip_blocked & all) == all) break;  // nothing later can commute forward
    }
  }
  p.qmask = pad_tile(q, pp.n, pp.k);
  return p;
}

// The pass that takes the most gates among the plain greedy one (its tile grows
// with the gate order: layer by layer, a strip of the circuit per pass) and the
// greedy passes restricted to a window of qubits contiguous in logical order
// (plus the forced low qubits).  On layered nearest-neighbour circuits a fixed
// window holds a parallelogram of the circuit -- several layers deep, shifted by
// the light cone -- instead of one layer's strip: fewer HBM passes.
Pass plan_best_pass(const std::vector<GateShape>& shapes, std::vector<char>& done, const PlanParams& pp,
                    uint64_t forbidden_flip, const std::vector<int>* l2p) {
  std::vector<char> best_done = done;
  Pass best = plan_one_pass(shapes, best_done, pp, forbidden_flip);
  if (pp.windows && !best.items.empty()) {
    int nq = 0;  // qubits in logical order (physical positions through l2p)
    for (const GateShape& s : shapes)
      if (s.touch) nq = std::max(nq, 64 - __builtin_clzll(s.touch));
    if (l2p) nq = static_cast<int>(l2p->size());
    auto phys = [&](int q) { return l2p ? (*l2p)[q] : q; };
    uint64_t seen = 0;
    for (int a = 0; a < nq; ++a) {
      uint64_t w = low_mask(pp.b);
      for (int q = a; q < nq && popc(w) < pp.k; ++q) {
        const uint64_t bit = 1ull << phys(q);
        if (!(bit & forbidden_flip)) w |= bit;
      }
      if (w == seen) continue;
      seen = w;
      std::vector<char> trial = done;
      Pass p = plan_one_pass(shapes, trial, pp, forbidden_flip, w);
      if (p.items.size() > best.items.size()) {
        best = std::move(p);
        best_done.swap(trial);
      }
    }
  }
  done.swap(best_done);
  return best;
}

std::vector<Pass> plan_gate_passes(const std::vector<GateShape>& shapes, const PlanParams& pp) {
  std::vector<char> done(shapes.size(), 0);
  std::vector<Pass> passes;
  size_t placed = 0;
  while (placed < shapes.size()) {
    Pass p = plan_best_pass(shapes, done, pp, 0, nullptr);
    if (p.items.empty()) throw std::runtime_error("planner made no progress (gate flip set wider than tile)");
    placed += p.items.size();
    passes.push_back(std::move(p));
  }
  return passes;
}

uint64_t remap_mask(uint64_t m, const std::vector<int>& l2p) {
  uint64_t r = 0;
  for (uint64_t v = m; v; v &= v - 1) r |= 1ull << l2p[__builtin_ctzll(v)];
  return r;
}

std::vector<Step> plan_schedule(const std::vector<GateShape>& logical, int n, int g, const PlanParams& pp,
                                std::vector<int>* l2p_final) {
  const int nloc = n - g;
  if (pp.n != nloc) throw std::runtime_error("plan_schedule: PlanParams.n must be the local qubit count");
  const int G = static_cast<int>(logical.size());
  std::vector<int> l2p(n), p2l(n);
  for (int q = 0; q < n; ++q) l2p[q] = p2l[q] = q;
  const uint64_t rank_mask = g ? (low_mask(n) & ~low_mask(nloc)) : 0;
  std::vector<GateShape> phys(G);
  auto refresh = [&]() {
    for (int i = 0; i < G; ++i) {
      phys[i] = logical[i];
      phys[i].flip = remap_mask(logical[i].flip, l2p);
      phys[i].touch = remap_mask(logical[i].touch, l2p);
    }
  };
  refresh();
  std::vector<char> done(G, 0);
  std::vector<Step> steps;
  int placed = 0, swaps_in_a_row = 0;
  while (placed < G) {
    std::vector<char> trial = done;
    Pass p = plan_best_pass(phys, trial, pp, rank_mask, &l2p);
    if (!p.items.empty()) {
      done.swap(trial);
      placed += static_cast<int>(p.items.size());
      Step st;
      st.pass = std::move(p);
      st.l2p = l2p;
      steps.push_back(std::move(st));
      swaps_in_a_row = 0;
      continue;
    }
    // the earliest pending gate flips a rank bit: swap it into a local position
    int gi = 0;
    while (done[gi]) ++gi;
    const uint64_t need = phys[gi].flip & rank_mask;
    if (!need || ++swaps_in_a_row > 2 * g + 2) throw std::runtime_error("sharded planner made no progress");
    const int pg = __builtin_ctzll(need);
    int best = -1, best_next = -1;
    for (int lp = nloc - 1; lp >= 0; --lp) {  // any local position; ties prefer high ones (contiguous halves)
      if ((phys[gi].flip >> lp) & 1) continue;
      int next = G;  // index of the next pending gate flipping this position
      for (int i = gi; i < G; ++i)
        if (!done[i] && ((phys[i].flip >> lp) & 1)) {
          next = i;
          break;
        }
      if (next > best_next) {
        best_next = next;
        best = lp;
      }
    }
    if (best < 0) throw std::runtime_error("a gate flips more qubits than a shard holds locally (use fewer shards)");
    Step st;
    st.swap = true;
    st.gbit = pg - nloc;
    st.lpos = best;
    st.l2p = l2p;
    steps.push_back(std::move(st));
    std::swap(p2l[pg], p2l[best]);
    l2p[p2l[pg]] = pg;
    l2p[p2l[best]] = best;
    refresh();
  }
  if (l2p_final) *l2p_final = l2p;
  return steps;
}

std::vector<Pass> plan_term_passes(const std::vector<uint64_t>& term_flips, const PlanParams& pp,
                                   std::vector<int>* direct) {
  // Greedy packing of flip masks into tiles: a pass is seeded with the widest
  // remaining mask and then takes, one at a time, the term that adds the fewest
  // new tile qubits (first in term order among equals) until nothing fits.  On
  // random Pauli sums this needs ~20 % fewer passes than first fit in term order
  // (cfg 5: 12 instead of 15 at n = 33; every pass but the first moves 3 S).
  const uint64_t low = low_mask(pp.b);
  std::vector<int> rem;
  for (int t = 0; t < static_cast<int>(term_flips.size()); ++t) {
    if (popc(low | term_flips[t]) > pp.k)
      direct->push_back(t);  // too wide for a tile: untiled gather pass
    else
      rem.push_back(t);
  }
  std::vector<Pass> passes;
  while (!rem.empty()) {
    size_t seed = 0;
    for (size_t i = 1; i < rem.size(); ++i)
      if (popc(term_flips[rem[i]] & ~low) > popc(term_flips[rem[seed]] & ~low)) seed = i;
    Pass p;
    uint64_t q = low | term_flips[rem[seed]];
    p.items.push_back(rem[seed]);
    rem.erase(rem.begin() + seed);
    while (static_cast<int>(p.items.size()) < pp.max_items) {
      int best = -1, best_add = 65;
      for (size_t i = 0; i < rem.size(); ++i) {
        const int total = popc(q | term_flips[rem[i]]);
        if (total > pp.k) continue;
        const int add = total - popc(q);
        if (add < best_add) {
          best_add = add;
          best = static_cast<int>(i);
          if (add == 0) break;
        }
      }
      if (best < 0) break;
      q |= term_flips[rem[best]];
      p.items.push_back(rem[best]);
      rem.erase(rem.begin() + best);
    }
    std::sort(p.items.begin(), p.items.end());  // term order inside a pass (summation order)
    p.qmask = pad_tile(q, pp.n, pp.k);
    passes.push_back(std::move(p));
  }
  return passes;
}

std::vector<Segment> plan_segments(const std::vector<uint32_t>& flip_pos, const std::vector<uint32_t>& touch_pos,
                                   const std::vector<char>& dense, int k, int regbits) {
  const uint32_t lanes = 31u;
  const uint32_t nonlane = ((k >= 32) ? ~0u : ((1u << k) - 1)) & ~lanes;
  const int m = static_cast<int>(flip_pos.size());
  // Dependencies inside the pass: i < j conflict when they share a tile
  // position that either of them flips (everything else commutes; positions
  // outside the tile are diagonal for every gate of the pass).
  std::vector<std::vector<int>> succ(m);
  std::vector<int> npred(m, 0);
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      const uint32_t shared = touch_pos[i] & touch_pos[j];
      if (shared & (flip_pos[i] | flip_pos[j])) {
        succ[i].push_back(j);
        ++npred[j];
      }
    }
  std::vector<char> done(m, 0);
  int remaining = m;
  // Gates runnable (transitively) with register set `regs`; `commit` applies them.
  auto closure = [&](uint32_t regs, std::vector<int>* order) {
    std::vector<int> pred = npred;
    std::vector<char> taken(done);
    int count = 0;
    bool progress = true;
    while (progress) {
      progress = false;
      for (int i = 0; i < m; ++i) {
        if (taken[i] || pred[i] != 0 || dense[i] || (flip_pos[i] & nonlane & ~regs)) continue;
        taken[i] = 1;
        ++count;
        progress = true;
        if (order) order->push_back(i);
        for (int j : succ[i]) --pred[j];
      }
    }
    return count;
  };
  auto retire = [&](const std::vector<int>& order) {
    for (int i : order) {
      done[i] = 1;
      --remaining;
      for (int j : succ[i]) --npred[j];
    }
  };
  std::vector<Segment> segs;
  while (remaining > 0) {
    // dense gates that are ready run as a shared-memory segment
    Segment sm;
    sm.reg = false;
    for (bool progress = true; progress;) {
      progress = false;
      for (int i = 0; i < m; ++i)
        if (!done[i] && dense[i] && npred[i] == 0) {
          sm.items.push_back(i);
          retire({i});
          progress = true;
          break;
        }
    }
    if (!sm.items.empty()) {
      segs.push_back(sm);
      continue;
    }
    // choose the register set greedily by how many gates it unlocks
    uint32_t regs = 0;
    int best_count = closure(0, nullptr);
    while (popc(regs) < regbits) {
      uint32_t cand_mask = 0;
      for (int i = 0; i < m; ++i)
        if (!done[i] && !dense[i]) cand_mask |= flip_pos[i] & nonlane & ~regs;
      if (!cand_mask) break;
      int best = -1, best_pos = -1;
      for (uint32_t v = cand_mask; v; v &= v - 1) {
        const int p = __builtin_ctz(v);
        const int c = closure(regs | (1u << p), nullptr);
        if (c > best) {
          best = c;
          best_pos = p;
        }
      }
      if (best <= best_count && popc(regs) > 0) {
        // no single position helps: take the flip set of the earliest pending gate
        for (int i = 0; i < m; ++i)
          if (!done[i] && !dense[i] && npred[i] == 0 && popc(regs | (flip_pos[i] & nonlane)) <= regbits &&
              (flip_pos[i] & nonlane & ~regs)) {
            regs |= flip_pos[i] & nonlane;
            break;
          }
        break;
      }
      regs |= 1u << best_pos;
      best_count = best;
    }
    Segment sg;
    sg.regmask = regs;
    closure(regs, &sg.items);
    if (sg.items.empty()) throw std::runtime_error("segment planner made no progress");
    retire(sg.items);
    segs.push_back(sg);
  }
  // Fill each register set to exactly `regbits` positions, preferring the
  // positions the following segments flip (fewer distinct layouts overall).
  for (size_t s = 0; s < segs.size(); ++s) {
    if (!segs[s].reg) continue;
    uint32_t& rm = segs[s].regmask;
    for (size_t t = s + 1; t < segs.size() && popc(rm) < regbits; ++t) {
      if (!segs[t].reg) continue;
      for (uint32_t v = segs[t].regmask & ~rm; v && popc(rm) < regbits; v &= v - 1) rm |= v & (~v + 1);
    }
    for (uint32_t v = nonlane & ~rm; v && popc(rm) < regbits; v &= v - 1) rm |= v & (~v + 1);
  }
  return segs;
}

std::vector<Segment> plan_segments_free(const std::vector<uint32_t>& flip_pos, const std::vector<uint32_t>& touch_pos,
                                        int k, int regbits, int lowb) {
  const int m = static_cast<int>(flip_pos.size());
  const uint32_t all = (k >= 32) ? ~0u : ((1u << k) - 1);
  const uint32_t low = (1u << lowb) - 1u;  // positions whose lanes keep global rows contiguous
  std::vector<std::vector<int>> succ(m);
  std::vector<int> npred(m, 0);
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      const uint32_t shared = touch_pos[i] & touch_pos[j];
      if (shared & (flip_pos[i] | flip_pos[j])) {
        succ[i].push_back(j);
        ++npred[j];
      }
    }
  // Gates runnable (transitively) from the state `done` whose flips lie in `regs`
  // (worklist over the conflict graph); returns how many, marks them in `taken`.
  auto closure = [&](const std::vector<char>& done, const std::vector<int>& pred0, uint32_t regs,
                     std::vector<char>* taken_out, std::vector<int>* order) {
    std::vector<int> pred = pred0;
    std::vector<char> taken = done;
    std::vector<int> ready;
    for (int i = m - 1; i >= 0; --i)
      if (!taken[i] && pred[i] == 0 && !(flip_pos[i] & ~regs)) ready.push_back(i);
    int count = 0;
    while (!ready.empty()) {
      // lowest index first: keeps the original gate order inside a segment
      const auto it = std::min_element(ready.begin(), ready.end());
      const int i = *it;
      ready.erase(it);
      taken[i] = 1;
      ++count;
      if (order) order->push_back(i);
      for (int j : succ[i])
        if (--pred[j] == 0 && !taken[j] && !(flip_pos[j] & ~regs)) ready.push_back(j);
    }
    if (taken_out) taken_out->swap(taken);
    return count;
  };
  // Beam search over sequences of register sets for the fewest segments (each
  // layout change is a shared-memory transpose of the whole tile): per state the
  // register sets -- every choice of `regbits` of the positions pending gates
  // flip -- are ranked by how many gates they run; the best few are expanded.
  struct Node {
    std::vector<char> done;
    int remaining = 0;
    std::vector<std::pair<uint32_t, std::vector<int>>> segs;  // (register set, items in order)
  };
  constexpr int kBeam = 6, kChildren = 4;
  std::vector<Node> beam(1);
  beam[0].done.assign(m, 0);
  beam[0].remaining = m;
  std::vector<Segment> segs;
  for (int depth = 0; depth < 4 * m + 4 && !beam.empty(); ++depth) {
    const Node* fin = nullptr;
    for (const Node& nd : beam)
      if (nd.remaining == 0) {
        fin = &nd;
        break;
      }
    if (fin) {
      for (const auto& sgp : fin->segs) {
        Segment sg;
        sg.regmask = sgp.first;
        sg.items = sgp.second;
        segs.push_back(std::move(sg));
      }
      break;
    }
    std::vector<Node> next;
    for (const Node& nd : beam) {
      std::vector<int> pred0(m, 0);
      uint32_t cand = 0;
      for (int i = 0; i < m; ++i) {
        if (nd.done[i]) continue;
        cand |= flip_pos[i] & all;
        for (int j : succ[i]) ++pred0[j];
      }
      std::vector<int> pos;
      for (uint32_t v = cand; v; v &= v - 1) pos.push_back(__builtin_ctz(v));
      const int np = static_cast<int>(pos.size());
      std::vector<std::pair<int, uint32_t>> ranked;  // (gates run, register set)
      if (np <= regbits) {
        ranked.push_back({closure(nd.done, pred0, cand, nullptr, nullptr), cand});
      } else {
        // every regbits-subset of the candidate positions (Gosper's hack)
        for (uint32_t c = (1u << regbits) - 1u; c < (1u << np);) {
          uint32_t regs = 0;
          for (uint32_t v = c; v; v &= v - 1) regs |= 1u << pos[__builtin_ctz(v)];
          // ties: keep the low positions free for the lanes
          ranked.push_back({closure(nd.done, pred0, regs, nullptr, nullptr) * 64 - popc(regs & low), regs});
          const uint32_t t = c | (c - 1);
          c = (t + 1) | (((~t & -~t) - 1) >> (__builtin_ctz(c) + 1));
        }
      }
      std::sort(ranked.begin(), ranked.end(), [](const auto& a, const auto& b) { return a.first > b.first || (a.first == b.first && a.second < b.second); });
      int kept = 0;
      std::vector<std::vector<char>> seen;
      for (const auto& rk : ranked) {
        if (kept >= kChildren) break;
        Node ch;
        ch.segs = nd.segs;
        std::vector<int> order;
        const int cnt = closure(nd.done, pred0, rk.second, &ch.done, &order);
        if (cnt == 0) break;
        if (std::find(seen.begin(), seen.end(), ch.done) != seen.end()) continue;  // same gates as a better-ranked set
        seen.push_back(ch.done);
        ch.remaining = nd.remaining - cnt;
        ch.segs.push_back({rk.second, std::move(order)});
        next.push_back(std::move(ch));
        ++kept;
      }
    }
    if (next.empty()) throw std::runtime_error("free-lane segment planner made no progress");
    std::stable_sort(next.begin(), next.end(), [](const Node& a, const Node& b) { return a.remaining < b.remaining; });
    // distinct states only
    std::vector<Node> pruned;
    for (Node& nd : next) {
      bool dup = false;
      for (const Node& q : pruned) dup = dup || q.done == nd.done;
      if (!dup) pruned.push_back(std::move(nd));
      if (static_cast<int>(pruned.size()) >= kBeam) break;
    }
    beam.swap(pruned);
  }
  if (m > 0 && segs.empty()) throw std::runtime_error("free-lane segment planner did not finish");
  // Fill register sets to `regbits` (positions the next segments flip first:
  // fewer distinct layouts), then lanes: 0..4 where free, else the lowest free
  // positions.  Equal consecutive layouts need no transpose.
  for (size_t s = 0; s < segs.size(); ++s) {
    uint32_t& rm = segs[s].regmask;
    for (size_t t = s + 1; t < segs.size() && popc(rm) < regbits; ++t)
      for (uint32_t v = segs[t].regmask & ~rm; v && popc(rm) < regbits; v &= v - 1) rm |= v & (~v + 1);
    for (uint32_t v = all & ~rm & ~low & ~31u; v && popc(rm) < regbits; v &= v - 1) rm |= v & (~v + 1);
    for (uint32_t v = all & ~rm & ~low; v && popc(rm) < regbits; v &= v - 1) rm |= v & (~v + 1);
    for (uint32_t v = all & ~rm; v && popc(rm) < regbits; v &= v - 1) rm |= v & (~v + 1);
    uint32_t lanes = 31u & ~rm;
    for (uint32_t v = all & ~rm & ~lanes; v && popc(lanes) < 5; v &= v - 1) lanes |= v & (~v + 1);
    segs[s].lanemask = lanes;
  }
  return segs;
}

double segment_plan_cost(const std::vector<Segment>& segs, const std::vector<uint32_t>& flip_pos, double lane_cost,
                         double xpose_cost, int lowb) {
  const uint32_t low = (1u << lowb) - 1u;
  double c = 0.0;
  uint32_t prev_r = ~0u, prev_l = ~0u;
  for (size_t s = 0; s < segs.size(); ++s) {
    const Segment& sg = segs[s];
    if (!sg.reg) return 1e30;
    if (s > 0 && (sg.regmask != prev_r || sg.lanemask != prev_l)) c += xpose_cost;
    prev_r = sg.regmask;
    prev_l = sg.lanemask;
    for (int i : sg.items) {
      const uint32_t f = flip_pos[i];
      c += f == 0 ? 0.5 : ((f & sg.lanemask) ? lane_cost : 1.0);
    }
  }
  if (!segs.empty() && (segs.back().lanemask & low) != low) c += xpose_cost;   // forward store
  if (!segs.empty() && (segs.front().lanemask & low) != low) c += xpose_cost;  // reverse store
  return c;
}

int choose_tile_qubits(int n, int requested, int sms, int min_tiles_per_sm) {
  if (requested > 0) return std::min(requested, n);
  if (n <= 10) return n;  // whole state in one tile: one CTA, no HBM round trips between passes
  int k = std::min(n, 11);
  // keep at least a few tiles per SM so the persistent grid stays balanced
  while (k > 9 && (n - k) < 62 && (1ll << (n - k)) < int64_t(min_tiles_per_sm) * sms) --k;
  return std::min(k, n);
}

}  // namespace svgb
