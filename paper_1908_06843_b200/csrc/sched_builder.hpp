// Host-side builder of the balanced segment schedules the enumerators run
// (see SchedDesc / run_schedule in bsc_kernels.cuh). Shared by the BSC and the
// multi-valued (tsc/dsc) state templates.
#pragma once
#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "bsc_engine.hpp"
#include "bsc_kernels.cuh"

namespace bscgpu {

constexpr int kSlots = 2 * kSchedRuns;  // ≤ R−1 split outputs, ≤ 2R−2 partials

struct ScheduleBuilder {
  int zero_off = 0;   // byte offset of the zero slot (an empty list reads it)
  int part_base = 0;  // first split slot (doubles from the warp region base)
  std::vector<SchedDesc> sched;
  std::vector<uint32_t> ent;  // packed: src/8 | dst code << 16
  std::vector<int4> splits;

  static unsigned w16(int byte_off) {
    if (byte_off < 0 || byte_off / 8 > 0xffff) throw Error(kConfig, "gpu: state template exceeds the 16-bit table range");
    return static_cast<unsigned>(byte_off / 8);
  }

  // Balanced lane schedule of one pass: the lists (byte offsets of the values
  // to sum) of every output are concatenated in output order and cut into R
  // equal runs. An output whose list lies inside one run is written directly
  // by that lane; one that spans runs leaves a partial per run in consecutive
  // slots, summed afterwards.
  void add(const std::vector<std::vector<int>>& ls, const std::vector<int>& targets) {
    constexpr int R = kSchedRuns;
    std::vector<std::pair<int, int>> seq;  // (byte offset, output)
    for (size_t o = 0; o < ls.size(); ++o) {
      if (ls[o].empty()) seq.emplace_back(zero_off, static_cast<int>(o));  // writes 0
      for (int v : ls[o]) seq.emplace_back(v, static_cast<int>(o));
    }
    const int T = static_cast<int>(seq.size());
    const int iters = (T + R - 1) / R;
    std::vector<int> first_lane(ls.size(), 1 << 30), last_lane(ls.size(), -1);
    for (int j = 0; j < T; ++j) {
      const int o = seq[j].second, l = j / iters;
      first_lane[o] = std::min(first_lane[o], l);
      last_lane[o] = std::max(last_lane[o], l);
    }
    // dst: ≥ 0 output byte offset, −1 continue, ≤ −2 split slot −dst−2 (see seg_flush)
    auto pack = [&](int src, int dst) {
      uint32_t code = 0xffffu;
      if (dst >= 0) code = w16(dst);
      else if (dst <= -2) code = 0x8000u | static_cast<uint32_t>(part_base + (-dst - 2));
      if (dst != -1 && (code & 0x7fffu) >= 0x7fffu) throw Error(kConfig, "gpu: schedule destination out of range");
      if (dst >= 0 && code > 0x7fffu) throw Error(kConfig, "gpu: schedule destination out of range");
      return w16(src) | (code << 16);
    };
    // runs → list segments (the entries of one output inside one run)
    struct Seg {
      std::vector<int> src;
      int dst;
    };
    std::vector<std::vector<Seg>> runs(R);
    std::vector<int> slot_begin(ls.size(), -1);
    int slot = 0;
    for (int l = 0; l < R; ++l) {
      const int b = l * iters, e = std::min(T, b + iters);
      for (int j = b; j < e; ++j) {
        const int o = seq[j].second;
        if (j == b || seq[j - 1].second != o) runs[l].push_back(Seg{{}, -1});
        runs[l].back().src.push_back(seq[j].first);
        if (j + 1 == e || seq[j + 1].second != o) {
          if (first_lane[o] == last_lane[o]) {
            runs[l].back().dst = targets[o];
          } else {
            if (slot_begin[o] < 0) slot_begin[o] = slot;
            runs[l].back().dst = -(slot + 2);
            ++slot;
          }
        }
      }
    }
    // Emit one entry per run per iteration. Within a segment the order is
    // free (it is a sum), so each half-warp's 16 loads of one instruction are
    // picked greedily to fall in distinct 8-byte shared-memory banks.
    std::vector<uint32_t> rows(static_cast<size_t>(iters) * R, pack(zero_off, -1));
    std::vector<size_t> cur(R, 0);
    std::vector<std::vector<int>> rem(R);
    for (int l = 0; l < R; ++l)
      if (!runs[l].empty()) rem[l] = runs[l][0].src;
    for (int it = 0; it < iters; ++it)
      for (int u = 0; u < R / 32; ++u)
        for (int half = 0; half < 2; ++half) {
          unsigned used = 0;
          for (int k = 0; k < 16; ++k) {
            const int l = 32 * u + 16 * half + k;
            if (cur[l] >= runs[l].size()) continue;
            auto& r = rem[l];
            size_t pick = 0;
            for (size_t q = 0; q < r.size(); ++q)
              if (!((used >> ((r[q] / 8) & 15)) & 1u)) {
                pick = q;
                break;
              }
            const int src = r[pick];
            used |= 1u << ((src / 8) & 15);
            r[pick] = r.back();
            r.pop_back();
            const int dst = r.empty() ? runs[l][cur[l]].dst : -1;
            rows[static_cast<size_t>(it) * R + l] = pack(src, dst);
            if (r.empty() && ++cur[l] < runs[l].size()) r = runs[l][cur[l]].src;
          }
        }
    SchedDesc sd{iters, static_cast<int>(ent.size() / R), 0, static_cast<int>(splits.size())};
    for (size_t o = 0; o < ls.size(); ++o)
      if (first_lane[o] != last_lane[o]) {
        const int nparts = last_lane[o] - first_lane[o] + 1;
        splits.push_back(int4{targets[o], slot_begin[o], slot_begin[o] + nparts, 0});
        ++sd.n_split;
      }
    if (sd.n_split >= R || slot > kSlots) throw Error(kInternal, "state template: schedule split overflow");
    ent.insert(ent.end(), rows.begin(), rows.end());
    sched.push_back(sd);
  }
};

}  // namespace bscgpu
