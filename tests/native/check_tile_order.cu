// Host-side check that tile_order() is a bijection onto its trapezoid (run by tests).
#include <cstdio>
#include <set>
#include <utility>
#include "../../paper_2503_04424_b200/csrc/tile.cuh"
int main() {
  int bad = 0, cases = 0;
  for (int nt = 1; nt <= 24; ++nt)
    for (int j0 = 0; j0 < nt; ++j0)
      for (int j1 = j0 + 1; j1 <= nt; ++j1)
        for (int lower = 0; lower <= 1; ++lower)
          for (int row_off = 0; row_off <= 1; ++row_off)
            for (int i0 : {0, 3})
              for (int G : {1, 3, 8})
               for (int stride : {0, 2, 3})
                for (int off = 0; off < (stride > 1 ? stride : 1); ++off) {
                b2d::TileSet ts{i0, nt, j0, j1, lower, row_off, stride, off};
                std::set<std::pair<int, int>> want, got;
                const int st = stride > 1 ? stride : 1;
                for (int j = j0; j < j1; ++j)
                  for (int i = i0; i < nt; ++i)
                    if (!lower || i * st + off >= j + row_off) want.insert({i, j});
                if ((long)want.size() != ts.count()) ++bad;
                for (long b = 0; b < (long)want.size(); ++b) {
                  int i, j;
                  b2d::tile_order(b, ts, G, &i, &j);
                  got.insert({i, j});
                }
                ++cases;
                if (got != want) {
                  if (bad++ < 5) printf("mismatch nt=%d j0=%d j1=%d lower=%d off=%d i0=%d G=%d\n", nt, j0, j1, lower, row_off, i0, G);
                }
              }
  printf("%d cases, %d bad\n", cases, bad);
  return bad != 0;
}
