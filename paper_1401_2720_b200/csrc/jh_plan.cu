// The 4-cycle plan of a pivot table, used by engine 1 (jh_vpair.cu).
//
// For the reversed row-closest strategy (rrow, the Mantharam-Eberlein
// equivalent; reference strategy.py:377-419) the pairs of two consecutive
// p-steps close over groups of four block-columns: tasks t1 = (p1, q1), t2 =
// (p2, q2) of p-step s-1 and tasks u1, u2 of p-step s, each u taking one
// block-column from t1 and one from t2.  Engine 1 moves the four V
// block-columns of such a cycle through shared memory once and applies both
// p-steps' transforms.  The plan is built on the host and copied to the
// device; a table without the structure is rejected (engine 0 runs it).
#include "jh_kernels.h"

#include <vector>

namespace jh {

int64_t cycle_plan_ints(int b, int steps) {
  if (b < 4 || b % 4 || steps < 1) return 0;
  const int64_t S = steps, T = b / 2, nc = T / 2;
  return S * nc * 8 + 2 * S * T;
}

int cycle_plan(const int32_t *outer, int b, int steps, int32_t *plan) {
  if (b < 4 || b % 4 || steps < 1) return 1;
  const int S = steps, T = b / 2, nc = T / 2;
  int32_t *cyc = plan, *tpos = plan + (int64_t)S * nc * 8, *upos = tpos + (int64_t)S * T;
  for (int64_t i = 0; i < cycle_plan_ints(b, steps); i++) plan[i] = 0;
  std::vector<int> tprev(b), tcur(b), seen(T);
  auto pr = [&](int s, int t, int k) { return outer[((int64_t)s * T + t) * 2 + k]; };
  // boundary s joins p-steps sp = s-1 (s = 0: the wrap from the last p-step)
  auto boundary = [&](int s) -> bool {
    const int sp = (s + S - 1) % S;
    for (int t = 0; t < T; t++) {
      tprev[pr(sp, t, 0)] = t;
      tprev[pr(sp, t, 1)] = t;
      tcur[pr(s, t, 0)] = t;
      tcur[pr(s, t, 1)] = t;
      seen[t] = 0;
    }
    int c = 0;
    for (int t1 = 0; t1 < T; t1++) {
      if (seen[t1]) continue;
      const int p1 = pr(sp, t1, 0), q1 = pr(sp, t1, 1);
      const int u1 = tcur[p1], u2 = tcur[q1];
      if (u1 == u2) return false;  // same pair in both steps: not a 4-cycle
      const int x = pr(s, u1, 0) == p1 ? pr(s, u1, 1) : pr(s, u1, 0);
      const int y = pr(s, u2, 0) == q1 ? pr(s, u2, 1) : pr(s, u2, 0);
      const int t2 = tprev[x];
      if (tprev[y] != t2 || t2 == t1 || seen[t2]) return false;
      const int p2 = pr(sp, t2, 0), q2 = pr(sp, t2, 1);
      auto slot = [&](int col) {
        return col == p1 ? 0 : col == q1 ? 1 : col == p2 ? 2 : col == q2 ? 3 : -1;
      };
      if (c >= nc) return false;
      int32_t *e = cyc + ((int64_t)s * nc + c) * 8;
      e[0] = t1;
      e[1] = t2;
      e[2] = u1;
      e[3] = u2;
      e[4] = slot(pr(s, u1, 0));
      e[5] = slot(pr(s, u1, 1));
      e[6] = slot(pr(s, u2, 0));
      e[7] = slot(pr(s, u2, 1));
      for (int i = 4; i < 8; i++)
        if (e[i] < 0) return false;
      tpos[(int64_t)sp * T + t1] = 2 * c;
      tpos[(int64_t)sp * T + t2] = 2 * c + 1;
      upos[(int64_t)s * T + u1] = 2 * c;
      upos[(int64_t)s * T + u2] = 2 * c + 1;
      seen[t1] = seen[t2] = 1;
      c++;
    }
    return c == nc;
  };
  for (int s = 1; s < S; s++)
    if (!boundary(s)) return 1;
  // Boundary 0 is read only for a last p-step updated alone, which uses just
  // the grouping of its own tasks into pairs (t1, t2): the wrap's 4-cycles
  // when the table has them, any pairing otherwise (a table segment).
  if (S == 1 || !boundary(0)) {
    for (int c = 0; c < nc; c++) {
      int32_t *e = cyc + (int64_t)c * 8;
      e[0] = e[2] = 2 * c;
      e[1] = e[3] = 2 * c + 1;
      e[4] = 0, e[5] = 1, e[6] = 2, e[7] = 3;
    }
  }
  return 0;
}

}  // namespace jh
