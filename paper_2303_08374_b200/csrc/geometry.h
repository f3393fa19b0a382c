// Launch geometry shared by the kernels and by the host: how a message is
// split into shares, chunks and rounds. Pure integer functions of values every
// rank agrees on (byte counts, CTA counts, slot sizes), compiled for the
// device (kernels), the host (launchers) and plain C++ (tests/geometry_check.cpp
// proves byte coverage at p = 8 for the BASELINE sizes without a GPU).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define MCRDL_HD __host__ __device__ __forceinline__
#else
#define MCRDL_HD inline
#endif

namespace mcrdl {

MCRDL_HD int64_t gmin(int64_t a, int64_t b) { return a < b ? a : b; }
MCRDL_HD int64_t gmax(int64_t a, int64_t b) { return a > b ? a : b; }

// ------------------------------------------------ block-cooperative shares
// [s, e) share of `len` bytes for block b of G (16-byte aligned starts).
MCRDL_HD void byte_share(int64_t len, int b, int G, int64_t& s, int64_t& e) {
  int64_t chunk = (len + G - 1) / G;
  chunk = (chunk + 15) & ~int64_t(15);
  s = gmin(len, int64_t(b) * chunk);
  e = gmin(len, s + chunk);
}

// ------------------------------------------------ two-shot all_reduce (K2)
// The message is npk 16-byte packs; segment q (owned by rank q) is packs
// [q*sp, (q+1)*sp); share s of every segment is packs [rb, re) relative to
// the segment start with rb = sp*s/gp, re = sp*(s+1)/gp.
MCRDL_HD int64_t seg_len(int64_t npk, int64_t sp, int q, int64_t rb, int64_t re) {
  // packs of share [rb, re) that exist in segment q
  const int64_t hi = gmin(re, npk - int64_t(q) * sp);
  return hi > rb ? hi - rb : 0;
}
MCRDL_HD int nchunks(int64_t len, int64_t chp, int s) {
  int k = int((len + chp - 1) / chp);
  return (k == 0 && s == 0) ? 1 : k;  // share 0 always carries a flag (order check)
}

// Host: shares and flag chunk of one two-shot launch of npk packs.
//   base shares gp: one per 32 KiB of segment, <= gp_max (2/3 of the SM
//   budget's 2 CTAs/SM: 3 roles x gp); TMA geometry (tma_geo): gs <= tma_ctas
//   single-thread bulk-copy senders leave room for more reducer/gatherer
//   shares (gs + 2 * shares <= 2 CTAs per budgeted SM). chp (packs per flag
//   chunk) keeps every share at <= 4000 chunks (12-bit flag step) and at
//   least chunk_kb KiB. Every input is agreed by all ranks.
struct TwoShotGeo {
  int64_t sp;      // packs per segment (rank q owns [q*sp, (q+1)*sp))
  int64_t segb;    // workspace bytes per segment slot
  int64_t gp;      // base shares (NVLS roles use these)
  int64_t shares;  // shares of this launch (== gp unless tma_geo)
  int64_t chp;     // packs per flag chunk for `shares`
  int gs;          // TMA sender CTAs (tma_geo)
};
MCRDL_HD int64_t chunk_packs(int64_t sp, int64_t shares, int64_t chunk_kb) {
  int64_t chp = ((sp + shares - 1) / shares + 3999) / 4000;
  return chp < chunk_kb * 64 ? chunk_kb * 64 : chp;  // KiB -> 16-byte packs
}
MCRDL_HD TwoShotGeo two_shot_geo(int64_t npk, int world, int num_sms, int64_t chunk_kb,
                                 bool tma_geo, int64_t gp_env, int64_t tma_ctas, int max_blocks) {
  TwoShotGeo g{};
  g.sp = (npk + world - 1) / world;
  g.segb = (g.sp * 16 + 255) / 256 * 256;
  int64_t gp = (g.sp * 16 + (32 << 10) - 1) / (32 << 10);
  int64_t cap = gp_env > 0 ? gp_env : 2 * num_sms / 3;
  cap = gmax(1, gmin(cap, max_blocks));
  g.gp = gmax(1, gmin(gp, cap));
  g.shares = g.gp;
  g.gs = int(gmin(g.gp, tma_ctas));
  if (tma_geo) {
    const int64_t room = (2 * num_sms - g.gs) / 2;
    if (gp_env <= 0 && g.shares < room)
      g.shares = gmax(1, gmin(room, (g.sp * 16 + (32 << 10) - 1) / (32 << 10)));
  }
  g.chp = chunk_packs(g.sp, g.shares, chunk_kb);
  return g;
}

// ------------------------------------------------ exchange engine (K5-K8)
constexpr int64_t kMaxSteps = 4000;  // < 4096 (12-bit flag step)

MCRDL_HD int64_t rounds_for(int64_t bytes, int64_t slot) {
  return bytes <= slot ? 1 : (bytes + slot - 1) / slot;
}
// CTAs serving one pair: a function of the pair's byte count only.
MCRDL_HD int pair_ctas(int64_t bytes, int gmax_ctas, int64_t per_cta, int64_t wide_min) {
  if (wide_min > 0 && bytes >= wide_min) per_cta *= 4;
  int64_t g = (bytes + per_cta - 1) / per_cta;
  return int(g < 1 ? 1 : (g > gmax_ctas ? gmax_ctas : g));
}
MCRDL_HD int64_t pair_chunk(int64_t bytes, int g, int64_t chunk_min) {
  // (~4 smaller chunks per share for push / copy-out overlap measured WORSE
  // for mid-size pairs: p = 4 all_to_allv 16 MiB 275 vs 325 GB/s — the extra
  // flag round trips cost more than the overlap gains)
  int64_t per = (bytes + g - 1) / g;
  int64_t ch = (per + kMaxSteps - 1) / kMaxSteps;
  ch = (ch + 15) & ~int64_t(15);
  return ch > chunk_min ? ch : chunk_min;
}

// Share s of round t of a pair moving B bytes: [a, e) relative to the round,
// in n chunks of `ch` bytes. A 0-byte pair still carries one empty chunk on
// share 0 (its flag is the order check / barrier).
struct Span {
  int64_t a, e;
  int n;
};
MCRDL_HD Span span_of(int64_t B, int64_t slot, int g, int64_t ch, int64_t t, int s) {
  Span sp{0, 0, 0};
  if (s >= g || t >= rounds_for(B, slot)) return sp;
  const int64_t len = gmin(slot, B - t * slot);
  // Share boundaries come from round 0 (the longest) in EVERY round: CTA s
  // owns the same slot bytes each round, so the receiver's per-share ack of
  // round t frees exactly what sender CTA s overwrites in round t+1 (a
  // shorter last round must not shift shares onto bytes another receiver
  // CTA is still landing).
  int64_t chunk = (gmin(slot, B) + g - 1) / g;
  chunk = (chunk + 15) & ~int64_t(15);
  sp.a = gmin(len, int64_t(s) * chunk);
  sp.e = gmin(len, sp.a + chunk);
  sp.n = int((sp.e - sp.a + ch - 1) / ch);
  if (B == 0 && s == 0 && t == 0) sp.n = 1;
  return sp;
}

// Chain bcast (k_bcast_chain): one launch of nb bytes is cut into chunks of
// `ch` bytes; CTA b serves chunks b, b + g, ... and counts one flag step per
// chunk, so ch doubles until no CTA needs more than kMaxSteps steps.
struct ChainGeo {
  int64_t g;   // CTAs
  int64_t ch;  // chunk bytes
};
MCRDL_HD ChainGeo chain_geo(int64_t nb, int64_t chunk, int64_t ctas, int num_sms, int max_blocks) {
  int64_t g = (nb + chunk - 1) / chunk;
  g = gmax(1, gmin(g, gmin(ctas, int64_t(max_blocks))));
  g = gmax(1, gmin(g, int64_t(2) * num_sms));
  int64_t ch = chunk;
  while ((nb + ch * g - 1) / (ch * g) > kMaxSteps) ch *= 2;
  return ChainGeo{g, ch};
}

}  // namespace mcrdl
