// Exact comparison of two k-mer ranks over the same pool (host, rare path).
//
// V_a = sum_j C_aj / D_aj with D_aj = min(nk_a, nk_j) (Eq. 1 summed over the
// pool).  The device orders ranks by 128-bit
// fixed-point keys; when two keys are closer than the pool size the order is
// not certified and sa_partition asks this routine for the exact answer
// (DESIGN.md §4).  It groups each row's terms by denominator,
// delta_d = sum_{D_aj = d} C_aj - sum_{D_bj = d} C_bj, and returns the sign of
// sum_d delta_d / d, accumulated as one fraction N / Den with Den = lcm of the
// denominators seen so far, in a small arbitrary-precision integer.
#include <algorithm>
#include <cstdint>
#include <map>
#include <vector>

namespace sa {

namespace {

using u64 = uint64_t;
using u128 = unsigned __int128;

struct Big {            // magnitude, little-endian 64-bit limbs
  std::vector<u64> l;
  bool zero() const { return l.empty(); }
  void trim() { while (!l.empty() && l.back() == 0) l.pop_back(); }
};

void mul_small(Big& a, u64 m) {
  if (m == 0) { a.l.clear(); return; }
  u64 carry = 0;
  for (auto& x : a.l) {
    u128 t = (u128)x * m + carry;
    x = (u64)t;
    carry = (u64)(t >> 64);
  }
  if (carry) a.l.push_back(carry);
}

u64 mod_small(const Big& a, u64 d) {
  u128 r = 0;
  for (size_t i = a.l.size(); i-- > 0;) r = ((r << 64) | a.l[i]) % d;
  return (u64)r;
}

void div_small(Big& a, u64 d) {   // exact or floor division
  u128 r = 0;
  for (size_t i = a.l.size(); i-- > 0;) {
    u128 cur = (r << 64) | a.l[i];
    a.l[i] = (u64)(cur / d);
    r = cur % d;
  }
  a.trim();
}

int cmp_mag(const Big& a, const Big& b) {
  if (a.l.size() != b.l.size()) return a.l.size() < b.l.size() ? -1 : 1;
  for (size_t i = a.l.size(); i-- > 0;)
    if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
  return 0;
}

void add_mag(Big& a, const Big& b) {
  if (a.l.size() < b.l.size()) a.l.resize(b.l.size(), 0);
  u64 carry = 0;
  for (size_t i = 0; i < a.l.size(); ++i) {
    u128 t = (u128)a.l[i] + (i < b.l.size() ? b.l[i] : 0) + carry;
    a.l[i] = (u64)t;
    carry = (u64)(t >> 64);
  }
  if (carry) a.l.push_back(carry);
}

// signed accumulator N = s * |N|
struct SBig {
  int s = 0;   // -1, 0, +1
  Big m;
};

void sub_mag_exact(Big& a, const Big& b) {   // |a| >= |b|
  u64 borrow = 0;
  for (size_t i = 0; i < a.l.size(); ++i) {
    const u64 bi = i < b.l.size() ? b.l[i] : 0;
    const u64 ai = a.l[i];
    const u64 r1 = ai - bi;
    const u64 b1 = ai < bi ? 1 : 0;
    const u64 r2 = r1 - borrow;
    const u64 b2 = r1 < borrow ? 1 : 0;
    a.l[i] = r2;
    borrow = b1 | b2;
  }
  a.trim();
}

void sadd(SBig& acc, int s, const Big& v) {
  if (s == 0 || v.zero()) return;
  if (acc.s == 0) { acc.s = s; acc.m = v; return; }
  if (acc.s == s) { add_mag(acc.m, v); return; }
  const int c = cmp_mag(acc.m, v);
  if (c == 0) { acc.s = 0; acc.m.l.clear(); return; }
  if (c > 0) { sub_mag_exact(acc.m, v); return; }
  Big t = v;
  sub_mag_exact(t, acc.m);
  acc.m = t;
  acc.s = s;
}

u64 gcd64(u64 a, u64 b) {
  while (b) { u64 t = a % b; a = b; b = t; }
  return a;
}

}  // namespace

int exact_compare(const uint16_t* Ca, int32_t nka, const uint16_t* Cb, int32_t nkb, const int32_t* nk_pool,
                  int npool) {
  std::map<int64_t, int64_t> delta;   // d -> sum C_a - sum C_b over terms with that denominator
  for (int j = 0; j < npool; ++j) {
    const int64_t da = std::min<int64_t>(nka, nk_pool[j]);
    const int64_t db = std::min<int64_t>(nkb, nk_pool[j]);
    if (da > 0 && Ca[j]) delta[da] += Ca[j];
    if (db > 0 && Cb[j]) delta[db] -= Cb[j];
  }
  SBig N;          // sum so far = N / Den
  Big Den;
  Den.l.push_back(1);
  for (const auto& kv : delta) {
    const int64_t dv = kv.second;
    if (dv == 0) continue;
    const u64 d = (u64)kv.first;
    const u64 g = gcd64(mod_small(Den, d), d);   // gcd(Den, d)
    const u64 m = d / g;
    // N/Den + dv/d = (N*m + dv*(Den/g)) / (Den*m)
    if (m != 1) mul_small(N.m, m);
    Big t = Den;
    div_small(t, g);
    mul_small(t, (u64)(dv < 0 ? -dv : dv));
    sadd(N, dv < 0 ? -1 : 1, t);
    if (m != 1) mul_small(Den, m);
  }
  return N.s;
}

}  // namespace sa
