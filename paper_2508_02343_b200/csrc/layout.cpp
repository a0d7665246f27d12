// layout.cpp -- plan-time shared-memory slot layout of the reorder-quantize gather
// ("gather layout"; offline, host only).
//
// The R = 2 RQ kernel transposes each tile into 4-byte slots (the two rows' BF16
// values of one channel) and then gathers x_r[j] = X[perm[j]]: lane l of a warp loads,
// at step q, reordered position 32 kb + 16 h + q of its half block.  For a random
// permutation the 32 channels of one load fall into ~3.5 x as many bank wavefronts as
// needed.  The slot of a channel is free up to what the transpose can write cheaply:
// this layout permutes the eight 4-channel chunks (16 B) inside every 32-channel
// (128-byte) line, parity preserving (even chunks to even positions), which keeps the
// transpose's store instructions conflict free (rq.cu) and lets a local search move
// bank bits 3..4 of every chunk.  Nothing computed changes: only where a value sits in
// shared memory.  The result is packed one u32 per line: nibble c = position of chunk c.
#include <algorithm>
#include <cstdint>
#include <vector>

namespace mmx {

std::vector<uint32_t> gather_layout(int K, const int n[3], const int32_t* perm) {
  const int nlines = K / 32;
  std::vector<uint8_t> pos(K / 4);                 // chunk -> position in its line
  for (int c = 0; c < K / 4; ++c) pos[c] = (uint8_t)(c & 7);
  // the kernel's gather steps (rq.cu tile_chunks): chunk c, step q, lane l reads
  // reordered position 32 b + 16 (l & 1) + q of block b = 16 c + l / 2 (dead lanes past
  // the last block compute on the last block)
  std::vector<int32_t> steps;                       // [S][32]
  const int nbt = K / 32, nch = (nbt + 15) / 16;
  (void)n;
  for (int c = 0; c < nch; ++c)
    for (int q = 0; q < 16; ++q)
      for (int l = 0; l < 32; ++l) {
        const int b = std::min(16 * c + l / 2, nbt - 1);
        steps.push_back(perm[32 * b + 16 * (l & 1) + q]);
      }
  const int S = (int)steps.size() / 32;
  if (S == 0) return std::vector<uint32_t>(nlines, 0x76543210u);
  // steps touching each line
  std::vector<std::vector<int>> line_steps(nlines);
  for (int s = 0; s < S; ++s)
    for (int l = 0; l < 32; ++l) {
      auto& v = line_steps[steps[32 * s + l] >> 5];
      if (v.empty() || v.back() != s) v.push_back(s);
    }
  for (auto& v : line_steps) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  // wavefronts of one step = the largest number of DISTINCT channels in one bank
  auto step_cost = [&](int s) {
    int cnt[32] = {0};
    int seen[32];
    int ns = 0, best = 0;
    for (int l = 0; l < 32; ++l) {
      const int p = steps[32 * s + l];
      bool dup = false;
      for (int i = 0; i < ns; ++i) dup |= seen[i] == p;
      if (dup) continue;
      seen[ns++] = p;
      const int bank = (4 * pos[p >> 2] + (p & 3)) & 31;
      best = std::max(best, ++cnt[bank]);
    }
    return best;
  };
  std::vector<int> cost(S);
  for (int s = 0; s < S; ++s) cost[s] = step_cost(s);
  for (int sweep = 0; sweep < 4; ++sweep) {
    int changed = 0;
    for (int L = 0; L < nlines; ++L) {
      const auto& ls = line_steps[L];
      if (ls.empty()) continue;
      uint8_t* pl = &pos[8 * L];
      for (int a = 0; a < 8; ++a)
        for (int b = a + 2; b < 8; b += 2) {       // same parity: keeps the transpose conflict free
          int before = 0, after = 0;
          for (int s : ls) before += cost[s];
          std::swap(pl[a], pl[b]);
          std::vector<int> nc(ls.size());
          for (size_t i = 0; i < ls.size(); ++i) after += (nc[i] = step_cost(ls[i]));
          if (after < before) {
            for (size_t i = 0; i < ls.size(); ++i) cost[ls[i]] = nc[i];
            ++changed;
          } else {
            std::swap(pl[a], pl[b]);
          }
        }
    }
    if (!changed) break;
  }
  std::vector<uint32_t> out(nlines);
  for (int L = 0; L < nlines; ++L) {
    uint32_t w = 0;
    for (int c = 0; c < 8; ++c) w |= (uint32_t)pos[8 * L + c] << (4 * c);
    out[L] = w;
  }
  return out;
}

// Total gather wavefronts of a layout (diagnostics / tests): natural layout = nullptr.
long long gather_wavefronts(int K, const int n[3], const int32_t* perm, const uint32_t* layout) {
  (void)n;
  long long tot = 0;
  const int nbt = K / 32, nch = (nbt + 15) / 16;
  for (int c = 0; c < nch; ++c)
    for (int q = 0; q < 16; ++q) {
      int cnt[32] = {0}, seen[32], ns = 0, best = 0;
      for (int l = 0; l < 32; ++l) {
        const int b = std::min(16 * c + l / 2, nbt - 1);
        const int p = perm[32 * b + 16 * (l & 1) + q];
        bool dup = false;
        for (int i = 0; i < ns; ++i) dup |= seen[i] == p;
        if (dup) continue;
        seen[ns++] = p;
        const int ps = layout ? (int)((layout[p >> 5] >> (4 * ((p >> 2) & 7))) & 7) : ((p >> 2) & 7);
        best = std::max(best, ++cnt[(4 * ps + (p & 3)) & 31]);
      }
      tot += best;
    }
  return tot;
}

}  // namespace mmx
