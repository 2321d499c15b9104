// Host-side pass planner: groups the gate list into HBM passes over tiles.
//
// A pass owns a tile-qubit set Q (|Q| = k, always containing the lowest b
// qubits so every tile row is a contiguous run of 2^b amplitudes).  The
// state is cut into 2^(n-k) independent tiles of 2^k amplitudes (fixed
// values of the non-tile qubits); one CTA stages a tile in shared memory and
// applies every gate of the pass to it, so the pass moves each amplitude
// through HBM once instead of once per gate.
//
// Only the FLIP qubits of a gate (X/Y factors of a Pauli-form gate, targets
// of a dense-matrix gate) must lie in Q.  Z factors and controls are
// diagonal: their effect inside a tile is a per-tile constant computed from
// the tile base index, so RZ/RZZ/controls never constrain the tile.
//
// Gates may be pulled forward past earlier, excluded gates only when they
// commute with them: on every shared qubit both act diagonally.  This keeps
// the planned order a valid reordering of the reference's gate sequence
// (svgrad/gradients.py:149-150 forward, :158-168 reverse).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/svgrad_b200.h"

namespace svgb {

struct GateShape {
  uint64_t flip;   // qubits that must be in the tile
  uint64_t touch;  // every qubit the gate reads (targets, controls)
  int nderiv;
};

struct Pass {
  uint64_t qmask = 0;        // tile qubits (popcount == k)
  std::vector<int> items;    // gate (or term) indices in application order
};

struct PlanParams {
  int n = 0;
  int k = 10;                // tile qubits
  int b = 5;                 // forced contiguous low qubits
  int max_items = 256;       // gates per pass cap
  int max_derivs = 96;       // derivative slots per pass cap (shared-memory accumulators)
  int windows = 1;           // also try passes restricted to windows of contiguous qubits (plan_best_pass)
};

GateShape gate_shape(const svg_gate& g);

// Forward gate passes; the reverse sweep walks the same passes backwards.
std::vector<Pass> plan_gate_passes(const std::vector<GateShape>& shapes, const PlanParams& pp);

// One greedy pass over the not-yet-`done` gates (marks the gates it takes).
// Gates flipping a `forbidden_flip` position (a sharded qubit) are skipped and
// block their qubits like any other excluded gate.
// Only gates whose flips lie in `allowed_flip` are taken (the others block).
Pass plan_one_pass(const std::vector<GateShape>& shapes, std::vector<char>& done, const PlanParams& pp,
                   uint64_t forbidden_flip, uint64_t allowed_flip = ~0ull);
// The best of the plain greedy pass and the greedy passes over windows of qubits
// contiguous in logical order (l2p: logical -> physical, or null for the identity).
Pass plan_best_pass(const std::vector<GateShape>& shapes, std::vector<char>& done, const PlanParams& pp,
                    uint64_t forbidden_flip, const std::vector<int>* l2p);

// Observable passes: terms grouped so each pass's flip masks fit one tile.
// Terms whose flip mask cannot share a tile with the low qubits go to `direct`
// (handled by an untiled gather kernel).
std::vector<Pass> plan_term_passes(const std::vector<uint64_t>& term_flips, const PlanParams& pp,
                                   std::vector<int>* direct);

// Register segments of one pass (register-tile kernels).  Tile positions
// 0..4 are lanes; a segment picks `regbits` of the other positions as
// register bits (the rest are warp bits, which its gates may not flip).
// Dense-matrix gates form shared-memory segments of their own.
struct Segment {
  bool reg = true;
  std::vector<int> items;   // indices into the pass's item list
  uint32_t regmask = 0;     // tile positions held in registers (reg segments)
  uint32_t lanemask = 31;   // tile positions on the 32 lanes (free-lane plans; else 0..4)
};
// Gates may be reordered inside a pass (dependency-aware list scheduling):
// each segment takes the register set that unlocks the most pending gates.
std::vector<Segment> plan_segments(const std::vector<uint32_t>& flip_pos, const std::vector<uint32_t>& touch_pos,
                                   const std::vector<char>& dense, int k, int regbits);

// Free-lane register segments (circuit-specialised kernels only, no dense
// gates): any `regbits` tile positions may be register bits, and a segment's
// gates flip register positions only -- no lane flips (a lane flip is a warp
// shuffle of both buffers, ~3.7x a register op).  Lanes are 5 positions the
// segment does not flip, preferring tile positions 0..4 (the global layout).
// Layout changes go through shared memory (transposes).  `lowb`: tile positions
// 0..lowb-1 are the contiguous low qubits of a global tile row; a layout whose
// lanes include them loads and stores whole rows whatever its other lanes are.
std::vector<Segment> plan_segments_free(const std::vector<uint32_t>& flip_pos, const std::vector<uint32_t>& touch_pos,
                                        int k, int regbits, int lowb = 5);

// Relative cost of a segment plan in register-op units (nb buffers): register
// flips 1, lane flips `lane_cost`, diagonal ops 0.5, each layout change
// `xpose_cost`, plus a final transpose when the last segment's lanes do not
// include tile positions 0..lowb-1 (the store needs whole global rows).
double segment_plan_cost(const std::vector<Segment>& segs, const std::vector<uint32_t>& flip_pos, double lane_cost,
                         double xpose_cost, int lowb = 5);

// ---- sharded schedules (state split over 2^g ranks by its top g PHYSICAL qubits) ----
//
// The schedule tracks a logical -> physical qubit map.  Gates only flip local
// physical positions; when the next gates need a flip on a rank bit, a SWAP
// step exchanges that rank bit with a local position (a pairwise half-shard
// exchange between ranks r and r ^ 2^gbit), chosen as the local qubit whose
// next flip lies furthest ahead.  Diagonal factors and controls on rank bits
// never need a swap (the rank bits enter the kernels' sign/control tests).
struct Step {
  bool swap = false;
  int gbit = 0, lpos = 0;   // swap: rank bit gbit <-> local physical position lpos
  Pass pass;                // pass: items = gate indices, qmask over physical local positions
  std::vector<int> l2p;     // logical -> physical map in effect for this step's gates
};

uint64_t remap_mask(uint64_t m, const std::vector<int>& l2p);

// n total qubits, g rank bits (pp.n must be n - g); returns the forward schedule
// and the final map (the observable and the reverse sweep start from it).
std::vector<Step> plan_schedule(const std::vector<GateShape>& logical, int n, int g, const PlanParams& pp,
                                std::vector<int>* l2p_final);

// Tile size choice for n qubits on `sms` SMs (auto when requested == 0): the
// widest tile (<= 11 qubits) leaving >= min_tiles_per_sm tiles per SM.
int choose_tile_qubits(int n, int requested, int sms, int min_tiles_per_sm = 4);

}  // namespace svgb
