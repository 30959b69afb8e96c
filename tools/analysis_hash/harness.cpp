#include "analysis.hpp"
#include <cstdio>
#include <cstdint>
#include <vector>
using namespace pinla;
template <class T> static uint64_t h(const std::vector<T>& v) {
  uint64_t x = 1469598103934665603ull;
  const unsigned char* p = (const unsigned char*)v.data();
  for (size_t i = 0; i < v.size() * sizeof(T); ++i) { x ^= p[i]; x *= 1099511628211ull; }
  return x ^ v.size();
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int64_t n, nnz, nd, nb;
  fread(&n, 8, 1, f); fread(&nnz, 8, 1, f); fread(&nd, 8, 1, f); fread(&nb, 8, 1, f);
  std::vector<int64_t> ip(n + 1), ix(nnz), pm(n), tb(nb);
  fread(ip.data(), 8, n + 1, f); fread(ix.data(), 8, nnz, f); fread(pm.data(), 8, n, f);
  if (nb) fread(tb.data(), 8, nb, f);
  fclose(f);
  Analysis A;
  analyze_tiles(A, n, ip.data(), ix.data(), pm.data(), nd, nb ? tb.data() : nullptr, nb, 59);
  std::vector<int32_t> ft, st, selt;
  for (auto& t : A.factor_tasks) { ft.push_back(t.type); ft.push_back(t.id); ft.push_back(t.level); }
  for (auto& t : A.selinv_tasks) { selt.push_back(t.type); selt.push_back(t.id); }
  for (auto& t : A.solve_tasks) { st.push_back(t.type); st.push_back(t.id); st.push_back(t.level); }
#define P(x) printf("%-16s %016llx\n", #x, (unsigned long long)h(A.x));
  P(upd_a) P(upd_b) P(chunk_rng) P(chunk_tile) P(chunk_flags) P(last_chunk) P(grp_rng) P(grp_tile)
  P(chunk_grp_ptr) P(f_ndep) P(f_succ_ptr) P(f_succ) P(f_ready0) P(f_prio) P(f_order)
  P(s_pa) P(s_pb) P(s_mode) P(s_chunk_rng) P(s_chunk_tile) P(s_chunk_flags) P(s_last_chunk)
  P(s_ndep) P(s_succ_ptr) P(s_succ) P(s_ready0) P(s_order) P(s_grp_rng) P(s_grp_tile)
  P(s_tile_grp_ptr) P(s_grp_buf) P(s_hot) P(sg_lo) P(sg_hi) P(sg_line) P(sf_ptr) P(sb_ptr)
  printf("%-16s %016llx\n%-16s %016llx\n%-16s %016llx\n", "factor_tasks", (unsigned long long)h(ft),
         "selinv_tasks", (unsigned long long)h(selt), "solve_tasks", (unsigned long long)h(st));
  return 0;
}
