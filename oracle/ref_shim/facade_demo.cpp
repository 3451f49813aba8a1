// Drop-in check (TEST INFRASTRUCTURE): the reference's own pipeline pieces vs
// neardup::b200 (include/neardup_b200.hpp) on the same inputs, in the
// reference's types.  Built by oracle/Makefile against the reference sources
// in place; run by tests/test_gpu_facade.py on the GPU box.
#include <unistd.h>

#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <vector>

#include "neardup/pipeline.hpp"
#include "neardup/synthetic.hpp"
#include "neardup_b200.hpp"

namespace {
std::string slurp(const std::filesystem::path& p) {
  std::ifstream f(p, std::ios::binary);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// every file of two workspaces, byte for byte (timings.json excepted)
bool same_workspace(const std::string& a, const std::string& b) {
  namespace fs = std::filesystem;
  std::map<std::string, std::string> fa, fb;
  for (auto* pr : {&a, &b})
    for (const auto& e : fs::recursive_directory_iterator(*pr))
      if (e.is_regular_file() && e.path().filename() != "timings.json")
        (pr == &a ? fa : fb)[fs::relative(e.path(), *pr).string()] = slurp(e.path());
  if (fa.size() != fb.size()) return std::printf("FAIL workspace file sets %zu vs %zu\n", fa.size(), fb.size()), false;
  for (const auto& [k, v] : fa) {
    auto it = fb.find(k);
    if (it == fb.end() || it->second != v) return std::printf("FAIL workspace file %s\n", k.c_str()), false;
  }
  return true;
}
}  // namespace

using namespace neardup;

int main() {
  SyntheticSpec spec;
  spec.doc_count = 3000;
  spec.group_count = 200;
  spec.group_size_max = 3;
  spec.seed = 21;
  SyntheticCorpus corpus = generate_synthetic(spec, 5, ShingleUnit::kByte);
  std::vector<CleanDocument> docs;
  for (size_t i = 0; i < corpus.texts.size(); ++i)
    docs.push_back({i * 2 + 7, corpus.texts[i], corpus.texts[i].size()});
  docs.push_back({99999, "abc", 3});  // too short: reported, skipped
  HashFamily fam = derive_family(5, 128, 5, ShingleUnit::kByte);
  b200::Device dev(0);

  std::vector<uint64_t> short_ref, short_gpu;
  auto ref = signature_batch(docs, fam, [&](uint64_t d) { short_ref.push_back(d); });
  auto gpu = b200::signature_batch(dev, docs, fam, [&](uint64_t d) { short_gpu.push_back(d); });
  if (ref.size() != gpu.size() || short_ref != short_gpu) return std::puts("FAIL batch shape"), 1;
  for (size_t i = 0; i < ref.size(); ++i)
    if (ref[i].doc_id != gpu[i].doc_id || ref[i].values != gpu[i].values)
      return std::printf("FAIL signature %zu\n", i), 1;

  const uint32_t K = choose_bucket_count(ref.size(), Ratio(2, 1));
  std::map<std::pair<uint32_t, uint32_t>, GatheredBucket> cells;
  for (const auto& s : ref) {
    auto a = band_bucket_ids(s.values, 16, 8, K);
    auto b = b200::band_bucket_ids(dev, s.values, 16, 8, K);
    if (a != b) return std::puts("FAIL band ids"), 1;
    for (uint32_t j = 0; j < 16; ++j) {
      auto& c = cells[{j, a[j]}];
      c.key = {j, a[j]};
      c.doc_ids.push_back(s.doc_id);
      c.signatures.insert(c.signatures.end(), s.values.begin(), s.values.end());
    }
  }
  GatherResult gathered;
  for (auto& [k, c] : cells)
    if (c.doc_ids.size() >= 2) gathered.buckets.push_back(std::move(c));
  SimilarityThreshold thr{Ratio(4, 5)};
  auto pr = compare_pass(gathered, 128, thr);
  auto pg = b200::compare_pass(dev, gathered, 128, thr);
  if (pr != pg) return std::printf("FAIL pairs %zu vs %zu\n", pr.size(), pg.size()), 1;

  UnionFind uf = union_pairs(pr);
  auto gr = components(uf);
  auto gg = b200::union_components(dev, pg);
  if (gr.size() != gg.size()) return std::puts("FAIL groups"), 1;
  for (size_t i = 0; i < gr.size(); ++i)
    if (gr[i].representative != gg[i].representative || gr[i].members != gg[i].members)
      return std::puts("FAIL group members"), 1;
  // whole in-memory dedup vs the reference's union of the same pairs
  std::vector<CleanDocument> clean(docs.begin(), docs.end() - 1);
  RunConfig cfg;
  uint64_t cand = 0;
  DedupReport rep = b200::dedup_in_memory(dev, clean, cfg, &cand);
  // the same through one context over three shards (nd_ctx_create_multi; on a
  // one-GPU box the shards share device 0)
  const int devs[3] = {0, 0, 0};
  b200::Device multi(std::span<const int>(devs, 3));
  if (multi.shards() != 3) return std::puts("FAIL shard count"), 1;
  uint64_t cand_m = 0;
  DedupReport rep_m = b200::dedup_in_memory(multi, clean, cfg, &cand_m);
  if (cand_m != cand || rep_m.groups.size() != rep.groups.size() ||
      rep_m.removals != rep.removals || rep_m.near_duplicates != rep.near_duplicates)
    return std::puts("FAIL multi-device dedup"), 1;
  for (size_t i = 0; i < rep.groups.size(); ++i)
    if (rep.groups[i].representative != rep_m.groups[i].representative ||
        rep.groups[i].members != rep_m.groups[i].members)
      return std::puts("FAIL multi-device groups"), 1;
  auto gm = b200::signature_batch(multi, docs, fam);
  for (size_t i = 0; i < gm.size(); ++i)
    if (gm[i].values != gpu[i].values) return std::puts("FAIL multi-device signatures"), 1;

  // the staged workflow: reference run_dedup vs b200::run_dedup, whole workspaces
  namespace fs = std::filesystem;
  const fs::path tmp = fs::temp_directory_path() / ("nd_facade_" + std::to_string(::getpid()));
  fs::create_directories(tmp / "in");
  write_synthetic(corpus, (tmp / "in" / "corpus.jsonl").string(), (tmp / "truth.jsonl").string());
  RunConfig rc;
  rc.inputs = {(tmp / "in").string()};
  rc.memory_budget = 300000;  // several gather passes
  rc.workspace = (tmp / "ws_ref").string();
  fs::create_directories(rc.workspace);
  DedupReport want = run_dedup(rc);
  rc.workspace = (tmp / "ws_gpu").string();
  DedupReport got = b200::run_dedup(dev, rc);
  if (want.groups.size() != got.groups.size() || want.removals != got.removals)
    return std::puts("FAIL staged report"), 1;
  if (!same_workspace((tmp / "ws_ref").string(), (tmp / "ws_gpu").string())) return 1;
  fs::remove_all(tmp);
  std::printf("FACADE OK signatures=%zu pairs=%zu groups=%zu\n", gpu.size(), pg.size(), gg.size());
  return 0;
}
