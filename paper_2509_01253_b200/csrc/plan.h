#pragma once
#include <cstdint>
#include <numeric>
#include <vector>

#include "sfhr_common.cuh"

namespace sfhr {

struct Plan {
  RingConst rc;
  int p_bits = 8, gamma = 0, beta = 1, pack_factor = 1;
  int shrink = 0;
  double bound_bits = 0, crt_bits = 0;
  std::vector<uint32_t> twid;                 // [np][M+1]
  std::vector<std::vector<uint32_t>> chains;  // stage0 chains (incl. leading 1)
  std::vector<std::vector<uint32_t>> reps_above;  // reps_above[j-1] = 1 + i t^j, i < t
  std::vector<int32_t> e1, e2, cvec;          // dual basis
  long long inv_m_mod_p = 0;
  uint64_t cu = 0;                            // centered M^-1 mod p as uint64
};

Plan make_plan(int t, int alpha, int p_bits, int D, int l, int gamma, int beta);
uint32_t inv_mod_M(const Plan& P, uint32_t d);

}  // namespace sfhr
