// Host-compiled check of the launch geometry in csrc/geometry.h (the exact
// functions the kernels and launchers use): every byte of every message is
// covered exactly once, by one share, one chunk and one round, and every
// flag step fits its 12-bit field — at p = 2, 4, 8 for the BASELINE sizes
// (cfg2 all_reduce sweep 8 B - 1 GiB, cfg3 DS-MoE, cfg4 DLRM uniform / Zipf,
// cfg1) and seeded random all_to_allv pairs. Needs no GPU.
//
//   g++ -O2 -std=c++17 -I paper_2303_08374_b200/csrc tests/geometry_check.cpp -o geometry_check
//   ./geometry_check            -> prints "OK <cases>" or the first violation
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "geometry.h"

using namespace mcrdl;

static int fail(const char* what, long long a, long long b, long long c) {
  std::printf("FAIL %s (%lld %lld %lld)\n", what, a, b, c);
  std::exit(1);
}

static const int kSms = 148;                        // B200 SM budget (one rank per GPU)
static const int64_t kHalf = int64_t(1) << 30;      // workspace half (2 GiB workspace)
static const int kMaxBlocks = 512;                  // flag slots per parity (common.cuh)
static long long g_cases = 0;

// Two-shot: one launch of npk packs at world p.
static void check_two_shot(int64_t npk, int p, int64_t chunk_kb, bool tma) {
  const TwoShotGeo g = two_shot_geo(npk, p, kSms, chunk_kb, tma, 0, 64, kMaxBlocks);
  if (g.sp * p < npk) fail("segments do not cover the message", npk, p, g.sp);
  const int ctas = tma ? g.gs + 2 * int(g.shares) : 3 * int(g.shares);
  if (ctas > 2 * kSms && !tma) fail("3 roles exceed 2 CTAs/SM", ctas, g.shares, npk);
  if (g.shares > kMaxBlocks) fail("more shares than flag slots", g.shares, npk, p);
  for (int q = 0; q < p; ++q) {
    int64_t covered = 0, expect_lo = 0;
    const int64_t seg = gmax(0, gmin(g.sp, npk - int64_t(q) * g.sp));
    for (int s = 0; s < g.shares; ++s) {
      const int64_t rb = g.sp * s / g.shares, re = g.sp * (s + 1) / g.shares;
      if (rb != expect_lo) fail("share gap / overlap", q, s, rb);
      expect_lo = re;
      const int64_t len = seg_len(npk, g.sp, q, rb, re);
      const int rows = nchunks(len, g.chp, s);
      if (rows > 4095) fail("flag step overflow (two-shot)", rows, npk, s);
      int64_t chunked = 0;
      for (int r = 0; r < rows; ++r) {
        const int64_t lo = int64_t(r) * g.chp;
        if (lo >= len) continue;
        chunked += gmin(g.chp, len - lo);
      }
      if (chunked != len) fail("chunks do not cover the share", chunked, len, s);
      covered += len;
    }
    if (expect_lo != g.sp) fail("shares do not end at the segment end", expect_lo, g.sp, q);
    if (covered != seg) fail("segment packs not covered exactly once", covered, seg, q);
  }
  ++g_cases;
}

// all_reduce of `bytes` at world p, as ar_typed chunks it into launches.
static void check_all_reduce(int64_t bytes, int esize, int p) {
  const int64_t n = (bytes + esize - 1) / esize;
  const int64_t N = 16 / esize;
  const int64_t room = kHalf / 2;
  const int64_t chunk_elems = ((room - int64_t(p) * 1024) / esize) / (int64_t(p) * 4 * N) * (int64_t(p) * 4 * N);
  int64_t done = 0;
  while (done < n) {
    const int64_t m = gmin(n - done, chunk_elems);
    const int64_t npk = (m + N - 1) / N;
    const int64_t chunk_kb = (p >= 4 && m * esize < (int64_t(128) << 20)) ? 128 : 256;
    const TwoShotGeo g = two_shot_geo(npk, p, kSms, chunk_kb, false, 0, 64, kMaxBlocks);
    // the launch's workspace footprint: p RS slots + p AG slots in one half
    if (2 * int64_t(p) * g.segb > kHalf) fail("two-shot launch exceeds a workspace half", m, p, g.segb);
    check_two_shot(npk, p, chunk_kb, false);
    check_two_shot(npk, p, chunk_kb, true);
    done += m;
  }
}

// Exchange pair of B bytes at world p: shares x chunks x rounds.
static void check_pair(int64_t B, int p) {
  const int64_t slot = kHalf / p / 256 * 256;
  const int g = pair_ctas(B, kSms, 32 << 10, int64_t(8) << 20);
  const int64_t ch = pair_chunk(B, g, 128 << 10);
  const int64_t R = rounds_for(B, slot);
  std::vector<int64_t> steps(g, 0);  // flag steps per share over all rounds
  int64_t covered = 0;
  for (int64_t t = 0; t < R; ++t) {
    int64_t expect = 0;
    const int64_t len = gmin(slot, B - t * slot);
    for (int s = 0; s < g; ++s) {
      const Span sp = span_of(B, slot, g, ch, t, s);
      if (sp.e > sp.a && sp.a != expect) fail("pair share gap / overlap", B, t, s);
      if (sp.e > sp.a) expect = sp.e;
      if (sp.e - sp.a > slot) fail("share beyond the slot", B, t, s);
      int64_t chunked = 0;
      for (int r = 0; r < sp.n; ++r) {
        const int64_t lo = sp.a + r * ch, hi = gmin(sp.e, lo + ch);
        if (hi > lo) chunked += hi - lo;
      }
      if (chunked != sp.e - sp.a) fail("pair chunks do not cover the share", B, t, s);
      steps[s] += sp.n;
      covered += sp.e - sp.a;
    }
    if (B > 0 && expect != len) fail("round not covered", B, t, expect);
  }
  if (covered != B) fail("pair bytes not covered exactly once", B, covered, p);
  for (int s = 0; s < g; ++s)
    if (steps[s] > 4095) fail("flag step overflow (exchange)", B, s, steps[s]);
  if (B == 0 && steps[0] != 1) fail("0-byte pair must carry one flag", B, steps[0], 0);
  ++g_cases;
}

// Chain bcast launch of nb bytes: chunks cover [0, nb) exactly once, CTA
// shares are disjoint, flag steps fit 12 bits, CTAs fit the flag slots.
static void check_chain(int64_t nb, int num_sms) {
  const ChainGeo geo = chain_geo(nb, 128 << 10, 128, num_sms, kMaxBlocks);
  if (geo.g < 1 || geo.g > kMaxBlocks || geo.g > 2 * num_sms) fail("chain CTAs", nb, geo.g, num_sms);
  const int64_t nch = (nb + geo.ch - 1) / geo.ch;
  int64_t covered = 0, expect = 0;
  for (int64_t j = 0; j < nch; ++j) {  // chunk j belongs to CTA j % g, step j / g + 1
    const int64_t lo = j * geo.ch, hi = gmin(nb, lo + geo.ch);
    if (lo != expect || hi <= lo) fail("chain chunk gap / overlap", nb, j, lo);
    expect = hi;
    covered += hi - lo;
    if (j / geo.g + 1 > 4095) fail("flag step overflow (chain)", nb, j, geo.g);
  }
  if (covered != nb) fail("chain bytes not covered exactly once", nb, covered, geo.ch);
  ++g_cases;
}

int main() {
  // chain bcast: one launch is at most a workspace half; co-located budgets too
  for (int sms : {148, 18, 4})
    for (int64_t nb : {int64_t(1), int64_t(4095), int64_t(128) << 10, (int64_t(128) << 10) + 1,
                       int64_t(300007), int64_t(64) << 20, (int64_t(1) << 30) - 3, kHalf,
                       int64_t(4) << 30})
      check_chain(nb, sms);
  for (int p : {2, 4, 8}) {
    // cfg2: all_reduce sweep 8 B - 1 GiB, f32 and bf16 (+ odd sizes)
    for (int k = 3; k <= 30; ++k)
      for (int es : {4, 2}) {
        check_all_reduce(int64_t(1) << k, es, p);
        check_all_reduce((int64_t(1) << k) + 4, es, p);
      }
    // cfg3: 4096 x 4096 bf16 tokens per rank, block per peer
    check_pair(int64_t(4096) * 4096 * 2 / p, p);
    // cfg4: DLRM 26 tables x 128, batch 65536, uniform and Zipf(1.1)
    std::vector<int> tables(p);
    for (int i = 0; i < p; ++i) tables[i] = 26 / p + (i < 26 % p ? 1 : 0);
    std::vector<int64_t> bu(p, 65536 / p), bz(p);
    double wsum = 0;
    for (int j = 0; j < p; ++j) wsum += std::pow(j + 1.0, -1.1);
    int64_t acc = 0;
    for (int j = 0; j < p; ++j) acc += bz[j] = int64_t(65536 * std::pow(j + 1.0, -1.1) / wsum);
    bz[p - 1] += 65536 - acc;
    for (const auto* b : {&bu, &bz})
      for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) check_pair((*b)[j] * tables[i] * 128 * 4, p);
    // cfg1 and seeded random pairs (0 bytes, odd sizes, multi-round)
    check_pair(262144 * 4 / 2, p);
    std::mt19937_64 rng(1234 + p);
    for (int i = 0; i < 2000; ++i) check_pair(int64_t(rng() % (int64_t(3) << 30)) >> (rng() % 31), p);
    for (int64_t B : {int64_t(0), int64_t(1), int64_t(15), int64_t(17), kHalf / p, kHalf / p + 1,
                      int64_t(3) * (kHalf / p) - 7})
      check_pair(B, p);
  }
  std::printf("OK %lld\n", g_cases);
  return 0;
}
