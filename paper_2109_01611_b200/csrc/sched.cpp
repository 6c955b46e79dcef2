// Native scheduler of the serving path: the paper's Algorithm 1
// "ElasticPartitioning" + FindBestFit (text P:566-598), the
// SBP whole-GPU temporal-sharing baseline, the ideal
// fixed-layout enumerator and the OLS fit of the interference model
// (P:638-652), under the readings listed in DESIGN.md §2.
//
// Integer microseconds / req/s / per-mille factors throughout; the knee and the
// interference factor use IEEE double in a fixed operation order (this TU is
// compiled with -ffp-contract=off) so plans are byte-identical to the oracle's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gpulet.h"

namespace {

constexpr int kGrid[6] = {20, 40, 50, 60, 80, 100};
// SMs per grid size when the caller gives none: the exact shares of 148 SMs in
// SM pairs (runtime.cpp sm_for_pct); the plan dump prints in.sm_count otherwise.
constexpr int kSm[6] = {30, 60, 74, 88, 118, 148};
constexpr int kStatB[6] = {1, 2, 4, 8, 16, 32};
constexpr int kBmax = 32;
constexpr double kEps = 1e-9;

int gidx(int p) {
  for (int i = 0; i < 6; ++i)
    if (kGrid[i] == p) return i;
  return -1;
}

struct Lane {
  int m;
  int64_t r;
};
struct Rec {
  int m;
  int64_t r;
  int b;
  int64_t e;
  int F;
};
struct GL {
  int gpu, slot, size;
  std::vector<Lane> lanes;
  int state;  // 0 remain, 1 alloc, 2 dead
};
struct Agg {
  bool some;
  double l2, mem;
};

class Sched {
 public:
  Sched(const gl_sched_input& in, int mode) : in(in), use_int(mode == 1) {}
  const gl_sched_input& in;
  bool use_int;
  bool fixed = false;
  std::vector<GL> pool;
  std::vector<int> alloc;  // insertion order

  int64_t L(int m, int b, int p) const { return in.lat_us[((size_t)m * 32 + (b - 1)) * 6 + gidx(p)]; }
  int sidx(int b) const {
    for (int i = 0; i < 6; ++i)
      if (kStatB[i] >= b) return i;
    return 5;
  }
  double l2(int m, int b, int p) const { return in.l2[((size_t)m * 6 + sidx(b)) * 6 + gidx(p)]; }
  double mem(int m, int b, int p) const { return in.mem[((size_t)m * 6 + sidx(b)) * 6 + gidx(p)]; }
  int64_t leff(int m, int b, int p, int F) const { return (L(m, b, p) * F + 999) / 1000; }

  int bsat(int m, int p) const {
    int best = 0;
    for (int b = 1; b <= kBmax; ++b)
      if (2 * L(m, b, p) <= in.slo_us[m]) best = b;
    return best;  // 0 = none
  }
  int64_t cap(int m, int p) const {
    const int b = bsat(m, p);
    if (!b) return 0;
    return (int64_t)b * 1000000 / leff(m, b, p, 1000);
  }
  void curve(int m, int64_t* r) const {
    for (int gi = 0; gi < 6; ++gi) {
      int64_t best = 0;
      for (int b = 1; b <= kBmax; ++b) {
        const int64_t l = L(m, b, kGrid[gi]);
        if (2 * l <= in.slo_us[m]) best = std::max(best, (int64_t)b * 1000000 / l);
      }
      r[gi] = best;
    }
  }
  // MaxEfficientPartition: knee of the normalised capacity curve; 0 = infeasible.
  int knee(int m) const {
    int64_t r[6];
    curve(m, r);
    int64_t rmax = 0;
    for (int i = 0; i < 6; ++i) rmax = std::max(rmax, r[i]);
    if (rmax == 0) return 0;
    double x[6], y[6], kap[6];
    for (int i = 0; i < 6; ++i) {
      x[i] = ((double)kGrid[i] - 20.0) / 80.0;
      y[i] = (double)r[i] / (double)rmax;
    }
    bool any = false;
    double kmax = 0;
    for (int i = 1; i < 5; ++i) {
      const double h1 = x[i] - x[i - 1];
      const double h2 = x[i + 1] - x[i];
      const double s1 = (y[i] - y[i - 1]) / h1;
      const double s2 = (y[i + 1] - y[i]) / h2;
      const double ypp = 2.0 * (s2 - s1) / (h1 + h2);
      const double yp = (y[i + 1] - y[i - 1]) / (h1 + h2);
      const double q = 1.0 + yp * yp;
      kap[i] = -ypp / (q * std::sqrt(q));
      if (r[i] > 0 && kap[i] > kEps) {
        kmax = any ? std::max(kmax, kap[i]) : kap[i];
        any = true;
      }
    }
    if (!any) return 100;
    for (int i = 1; i < 5; ++i)
      if (r[i] > 0 && kap[i] > kEps && kap[i] >= kmax - kEps) return kGrid[i];
    return 100;
  }
  int preq(int m, int64_t R) const {
    int64_t r[6];
    curve(m, r);
    for (int i = 0; i < 6; ++i)
      if (r[i] >= R) return kGrid[i];
    return 100;
  }

  int factor(int m, int b, int p, const Agg& A) const {
    if (!use_int || !A.some) return 1000;
    const double* c = in.coeffs;
    const double raw = ((((c[0] * l2(m, b, p)) + (c[1] * A.l2)) + (c[2] * mem(m, b, p))) + (c[3] * A.mem)) + c[4];
    const double f = std::ceil(1000.0 * raw);
    return f < 1000.0 ? 1000 : (int)f;
  }

  // Interference-aware batch (reading R13, P:532-537 / P:594): the largest
  // b <= b_sat with 2 Leff(b, F(b)) <= SLO, 0 if none; = b_sat without interference.
  int bint(int m, int p, const Agg& A) const {
    const int b0 = bsat(m, p);
    for (int b = b0; b >= 1; --b)
      if (2 * leff(m, b, p, factor(m, b, p, A)) <= in.slo_us[m]) return b;
    return 0;
  }

  // Interference-free batches of a lane set (for the partner aggregate).
  void batches(const std::vector<Lane>& lanes, int p, std::vector<int>& out) const {
    out.clear();
    if (lanes.size() == 1) {
      const int b = bsat(lanes[0].m, p);
      out.push_back(b ? b : 1);
      return;
    }
    int64_t D = -1;
    for (const Lane& ln : lanes) {
      const int b = bsat(ln.m, p);
      if (!b) {
        out.assign(lanes.size(), 1);
        return;
      }
      const int64_t d = leff(ln.m, b, p, 1000);
      D = D < 0 ? d : std::min(D, d);
    }
    for (const Lane& ln : lanes) {
      int64_t b = std::max<int64_t>(1, (ln.r * D + 999999) / 1000000);
      out.push_back((int)std::min<int64_t>(b, kBmax));
    }
  }
  Agg aggregate(int h) const {
    Agg A{false, 0, 0};
    if (h < 0 || pool[h].lanes.empty()) return A;
    std::vector<int> bs;
    batches(pool[h].lanes, pool[h].size, bs);
    for (size_t i = 0; i < bs.size(); ++i) {
      const double a = l2(pool[h].lanes[i].m, bs[i], pool[h].size);
      const double b = mem(pool[h].lanes[i].m, bs[i], pool[h].size);
      if (!A.some) {
        A.l2 = a, A.mem = b;
      } else {
        A.l2 = std::max(A.l2, a);
        A.mem = std::max(A.mem, b);
      }
      A.some = true;
    }
    return A;
  }

  // C2.6 lane-set feasibility; fills D and records.
  bool eval(const std::vector<Lane>& lanes, int p, const Agg& A, int64_t& D, std::vector<Rec>& recs) const {
    recs.clear();
    if (lanes.size() == 1) {
      const Lane& ln = lanes[0];
      const int b = bint(ln.m, p, A);
      if (!b) return false;
      const int F = factor(ln.m, b, p, A);
      const int64_t e = leff(ln.m, b, p, F);
      if (2 * e > in.slo_us[ln.m] || ln.r * e > (int64_t)b * 1000000) return false;
      D = e;
      recs.push_back(Rec{ln.m, ln.r, b, e, F});
      return true;
    }
    D = -1;
    for (const Lane& ln : lanes) {
      const int b = bint(ln.m, p, A);
      if (!b) return false;
      const int64_t d = leff(ln.m, b, p, factor(ln.m, b, p, A));
      D = D < 0 ? d : std::min(D, d);
    }
    int64_t tot = 0;
    for (const Lane& ln : lanes) {
      const int64_t b = std::max<int64_t>(1, (ln.r * D + 999999) / 1000000);
      if (b > kBmax) return false;
      const int F = factor(ln.m, (int)b, p, A);
      const int64_t e = leff(ln.m, (int)b, p, F);
      tot += e;
      recs.push_back(Rec{ln.m, ln.r, (int)b, e, F});
    }
    if (tot > D) return false;
    for (const Rec& r : recs)
      if (D + tot > in.slo_us[r.m]) return false;
    return true;
  }

  int sibling(int g) const {
    for (int i = 0; i < (int)pool.size(); ++i)
      if (pool[i].state != 2 && i != g && pool[i].gpu == pool[g].gpu && pool[i].slot != pool[g].slot) return i;
    return -1;
  }
  bool feasible(int g) const {
    int64_t D;
    std::vector<Rec> r;
    return eval(pool[g].lanes, pool[g].size, aggregate(sibling(g)), D, r);
  }
  bool sibling_ok(int g) const {
    const int h = sibling(g);
    if (h < 0 || pool[h].lanes.empty()) return true;
    int64_t D;
    std::vector<Rec> r;
    return eval(pool[h].lanes, pool[h].size, aggregate(g), D, r);
  }

  int add(int gpu, int slot, int size, int state) {
    pool.push_back(GL{gpu, slot, size, {}, state});
    return (int)pool.size() - 1;
  }

  std::vector<int> remain_sorted() const {
    std::vector<int> v;
    for (int i = 0; i < (int)pool.size(); ++i)
      if (pool[i].state == 0) v.push_back(i);
    std::sort(v.begin(), v.end(), [&](int a, int b) {
      if (pool[a].size != pool[b].size) return pool[a].size < pool[b].size;
      if (pool[a].gpu != pool[b].gpu) return pool[a].gpu < pool[b].gpu;
      return pool[a].slot < pool[b].slot;
    });
    return v;
  }

  bool try_merge(int ga, const Lane& ln) {
    pool[ga].lanes.push_back(ln);
    if (feasible(ga) && sibling_ok(ga)) return true;
    pool[ga].lanes.pop_back();
    return false;
  }
  bool hosts(int g, int m) const {
    for (const Lane& l : pool[g].lanes)
      if (l.m == m) return true;
    return false;
  }

  // FindBestFit scan at threshold p_ideal; returns assigned rate or -1.
  int64_t scan(int m, int pideal, int64_t R) {
    int chosen = -1, g_orig = -1, g_s = -1;
    int64_t r = 0;
    for (int g : remain_sorted()) {
      if (pool[g].state != 0 || pool[g].size < pideal) continue;
      int t = g, s = -1;
      bool split = false;
      if (pool[g].size == 100 && pideal < 100 && !fixed) {  // Split
        pool[g].state = 2;
        t = add(pool[g].gpu, 0, pideal, 0);
        s = add(pool[g].gpu, 1, 100 - pideal, 0);
        split = true;
      }
      const Agg A = aggregate(sibling(t));
      const int b = bint(m, pool[t].size, A);  // max b: 2 (L + intf) <= SLO
      bool ok = b > 0;
      int64_t e = 0;
      if (ok) {
        const int F = factor(m, b, pool[t].size, A);
        e = leff(m, b, pool[t].size, F);
      }
      if (ok) {
        r = std::min<int64_t>(R, (int64_t)b * 1000000 / e);
        pool[t].lanes = {Lane{m, r}};
        ok = sibling_ok(t);
        pool[t].lanes.clear();
      }
      if (!ok) {
        if (split) {
          pool[t].state = 2;
          pool[s].state = 2;
          pool[g].state = 0;
        }
        continue;
      }
      chosen = t;
      if (split) g_orig = g, g_s = s;
      break;
    }
    if (chosen < 0) return -1;
    for (int ga : alloc) {  // temporal merge
      if (hosts(ga, m)) continue;
      if (try_merge(ga, Lane{m, r})) {
        if (g_orig >= 0) {  // RevertSplit
          pool[chosen].state = 2;
          pool[g_s].state = 2;
          pool[g_orig].state = 0;
        }
        return r;
      }
    }
    pool[chosen].lanes = {Lane{m, r}};
    pool[chosen].state = 1;
    alloc.push_back(chosen);
    return r;
  }

  int64_t find_best_fit(int m, int pideal, int64_t R) {
    std::vector<int> th{pideal};
    std::vector<int> smaller;
    for (const GL& g : pool)
      if (g.state == 0 && g.size < pideal) smaller.push_back(g.size);
    std::sort(smaller.begin(), smaller.end(), std::greater<int>());
    smaller.erase(std::unique(smaller.begin(), smaller.end()), smaller.end());
    th.insert(th.end(), smaller.begin(), smaller.end());
    for (int t : th) {
      const int64_t r = scan(m, t, R);
      if (r >= 0) return r;
    }
    for (int ga : alloc) {  // E1: merge-only fallback
      if (hosts(ga, m)) continue;
      const int64_t c = cap(m, pool[ga].size);
      if (c <= 0) continue;
      const int64_t r = std::min(R, c);
      if (try_merge(ga, Lane{m, r})) return r;
    }
    return -1;
  }

  std::vector<int> order() const {
    std::vector<int> o;
    for (int m = 0; m < in.n_models; ++m)
      if (in.rates[m] > 0) o.push_back(m);
    std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return in.rates[a] > in.rates[b]; });
    return o;
  }

  bool run(const std::vector<std::vector<int>>* layout, int& failed) {
    pool.clear();
    alloc.clear();
    fixed = layout != nullptr;
    if (!layout) {
      for (int i = 0; i < in.num_gpus; ++i) add(i, 0, 100, 0);
    } else {
      for (int i = 0; i < (int)layout->size(); ++i)
        for (int s = 0; s < (int)(*layout)[i].size(); ++s) add(i, s, (*layout)[i][s], 0);
    }
    for (int m : order()) {
      const int pe = knee(m);
      if (!pe) {
        failed = m;
        return false;
      }
      int64_t R = in.rates[m];
      while (R > 0) {
        const int pideal = std::min(pe, preq(m, R));
        const int64_t r = find_best_fit(m, pideal, R);
        if (r < 0) {
          failed = m;
          return false;
        }
        R -= r;
      }
    }
    failed = -1;
    return true;
  }

  void dump(bool ok, int failed, std::string& out) const {
    std::vector<int> live;
    for (int i = 0; i < (int)pool.size(); ++i)
      if (pool[i].state != 2) live.push_back(i);
    std::sort(live.begin(), live.end(), [&](int a, int b) {
      if (pool[a].gpu != pool[b].gpu) return pool[a].gpu < pool[b].gpu;
      return pool[a].slot < pool[b].slot;
    });
    char buf[256];
    for (int g : live) {
      int64_t D = 0;
      std::vector<Rec> recs;
      if (!pool[g].lanes.empty()) eval(pool[g].lanes, pool[g].size, aggregate(sibling(g)), D, recs);
      snprintf(buf, sizeof buf, "{\"gpu\":%d,\"slot\":%d,\"size\":%d,\"sm\":%d,\"D_us\":%lld,\"lanes\":[", pool[g].gpu,
               pool[g].slot, pool[g].size, (in.sm_count ? in.sm_count[gidx(pool[g].size)] : kSm[gidx(pool[g].size)]), (long long)D);
      out += buf;
      for (size_t i = 0; i < recs.size(); ++i) {
        snprintf(buf, sizeof buf, "%s{\"model\":\"%s\",\"rate\":%lld,\"batch\":%d,\"exec_us\":%lld,\"F\":%d}",
                 i ? "," : "", in.names[recs[i].m], (long long)recs[i].r, recs[i].b, (long long)recs[i].e, recs[i].F);
        out += buf;
      }
      out += "]}\n";
    }
    out += "{\"verdict\":\"";
    out += ok ? "Schedulable" : "NotSchedulable";
    out += "\",\"failed_model\":";
    if (failed < 0) {
      out += "null";
    } else {
      out += "\"";
      out += in.names[failed];
      out += "\"";
    }
    out += "}\n";
  }
};

// SBP (Nexus squishy bin packing), reading C2.9, on bins of `size` %: whole GPUs
// (size 100, the temporal-sharing baseline) or the two halves of evenly split GPUs
// (size 50: "SBP algorithm that independently schedules two evenly split gpu-lets",
// Fig. success-case); num_gpus * 100 / size bins.
bool sbp(const gl_sched_input& in, std::string& out, int size = 100) {
  Sched S(in, 2);
  const int per = 100 / size, bins = in.num_gpus * per;
  std::vector<std::vector<Lane>> gpus;
  struct Resid {
    int m;
    int64_t r, e, D;
  };
  std::vector<Resid> resid;
  int failed = -1;
  for (int m : S.order()) {
    const int b = S.bsat(m, size);
    if (!b) {
      failed = m;
      break;
    }
    const int64_t L = S.L(m, b, size);
    const int64_t cap = (int64_t)b * 1000000 / L;
    const int64_t k = in.rates[m] / cap, r = in.rates[m] % cap;
    for (int64_t i = 0; i < k; ++i) gpus.push_back({Lane{m, cap}});
    if ((int)gpus.size() > bins) {
      failed = m;
      break;
    }
    if (r > 0) {
      const int64_t bp = (r * L + 999999) / 1000000;
      resid.push_back(Resid{m, r, S.L(m, (int)bp, size), L});
    }
  }
  if (failed < 0) {
    std::stable_sort(resid.begin(), resid.end(), [](const Resid& a, const Resid& b) { return a.e * b.D > b.e * a.D; });
    std::vector<std::vector<Lane>> rg;
    for (const Resid& x : resid) {
      int best = -1;
      int64_t bs = 0, bD = 1;
      for (int i = 0; i < (int)rg.size(); ++i) {
        std::vector<Lane> ls = rg[i];
        ls.push_back(Lane{x.m, x.r});
        int64_t D;
        std::vector<Rec> recs;
        if (!S.eval(ls, size, Agg{false, 0, 0}, D, recs)) continue;
        int64_t s = 0;
        for (const Rec& rc : recs) s += rc.e;
        if (best < 0 || s * bD > bs * D) best = i, bs = s, bD = D;
      }
      if (best < 0)
        rg.push_back({Lane{x.m, x.r}});
      else
        rg[best].push_back(Lane{x.m, x.r});
      if ((int)(gpus.size() + rg.size()) > bins) {
        failed = x.m;
        break;
      }
    }
    gpus.insert(gpus.end(), rg.begin(), rg.end());
  }
  for (int i = 0; i < bins; ++i) {
    const int id = S.add(i / per, i % per, size, 0);
    if (i < (int)gpus.size()) {
      S.pool[id].lanes = gpus[i];
      S.pool[id].state = 1;
    }
  }
  S.dump(failed < 0, failed, out);
  return failed < 0;
}

}  // namespace

extern "C" gl_status gl_schedule(const gl_sched_input* in, char* plan_buf, size_t cap, size_t* len, int32_t* verdict) {
  if (!in || !plan_buf || !len || !verdict || in->n_models < 1 || in->n_models > 8 || !in->lat_us || !in->slo_us ||
      !in->rates || !in->names || in->num_gpus < 1 || in->mode < 0 || in->mode > 4)
    return GL_E_ARG;
  if ((in->mode == 1) && (!in->l2 || !in->mem)) return GL_E_ARG;
  static const double zeros[8 * 36] = {0};
  gl_sched_input local = *in;
  if (!local.l2) local.l2 = zeros;
  if (!local.mem) local.mem = zeros;
  std::string out;
  bool ok;
  if (in->mode == 2 || in->mode == 4) {
    ok = sbp(local, out, in->mode == 2 ? 100 : 50);
  } else if (in->mode == 3) {
    // ideal: every multiset of per-GPU layouts {100}, {20,80}, {40,60}, {50,50}
    static const std::vector<int> L4[4] = {{100}, {20, 80}, {40, 60}, {50, 50}};
    if (in->num_gpus > 12) return GL_E_BUDGET;
    std::vector<int> idx(in->num_gpus, 0);
    ok = false;
    for (;;) {
      std::vector<std::vector<int>> lay;
      for (int i : idx) lay.push_back(L4[i]);
      Sched S(local, 1);
      int failed;
      ok = S.run(&lay, failed);
      out.clear();
      S.dump(ok, failed, out);
      if (ok) break;
      int k = in->num_gpus - 1;
      while (k >= 0 && idx[k] == 3) --k;
      if (k < 0) break;
      ++idx[k];
      for (int j = k + 1; j < in->num_gpus; ++j) idx[j] = idx[k];
    }
  } else {
    Sched S(local, in->mode);
    int failed;
    ok = S.run(nullptr, failed);
    S.dump(ok, failed, out);
  }
  if (out.size() + 1 > cap) return GL_E_BUDGET;
  std::memcpy(plan_buf, out.c_str(), out.size() + 1);
  *len = out.size();
  *verdict = ok ? 1 : 0;
  return GL_OK;
}

// OLS by Householder QR (interference model, "searched with linear regression").
extern "C" gl_status gl_fit_interference(const double* X, const double* y, int32_t n, double* c) {
  if (!X || !y || !c || n < 5) return GL_E_ARG;
  const int p = 5;
  std::vector<double> A(X, X + (size_t)n * p), b(y, y + n);
  double rmax = 0;
  for (int k = 0; k < p; ++k) {
    double norm = 0;
    for (int i = k; i < n; ++i) norm += A[(size_t)i * p + k] * A[(size_t)i * p + k];
    norm = std::sqrt(norm);
    const double akk = A[(size_t)k * p + k];
    const double alpha = akk > 0 ? -norm : norm;
    std::vector<double> v(n, 0.0);
    v[k] = akk - alpha;
    for (int i = k + 1; i < n; ++i) v[i] = A[(size_t)i * p + k];
    double vv = 0;
    for (int i = k; i < n; ++i) vv += v[i] * v[i];
    if (vv > 0) {
      for (int j = k; j < p; ++j) {
        double d = 0;
        for (int i = k; i < n; ++i) d += v[i] * A[(size_t)i * p + j];
        d = 2 * d / vv;
        for (int i = k; i < n; ++i) A[(size_t)i * p + j] -= d * v[i];
      }
      double d = 0;
      for (int i = k; i < n; ++i) d += v[i] * b[i];
      d = 2 * d / vv;
      for (int i = k; i < n; ++i) b[i] -= d * v[i];
    }
    rmax = std::max(rmax, std::fabs(A[(size_t)k * p + k]));
  }
  for (int k = 0; k < p; ++k)
    if (std::fabs(A[(size_t)k * p + k]) <= 1e-12 * rmax || rmax == 0) return GL_E_DATA;
  for (int k = p - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j < p; ++j) s -= A[(size_t)k * p + j] * c[j];
    c[k] = s / A[(size_t)k * p + k];
  }
  return GL_OK;
}
