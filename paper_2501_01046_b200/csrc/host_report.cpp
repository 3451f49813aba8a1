// Report writers for the union stage: groups.jsonl, removal.txt, summary.json,
// byte-identical with the reference's writers (pipeline.cpp:479-506, which
// format through nlohmann::ordered_json; the same header-only library is used
// here so numbers, in particular the ratio double, print identically).
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <unistd.h>
#include <vector>

#include <nlohmann/json.hpp>

#include "host_internal.hpp"

namespace ndb {
namespace {

// write_file_bytes (util.cpp:132-140): write, flush, optional fsync, close
void write_file(const std::string& path, const std::string& bytes, bool fsync_file) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(ND_ERR_IO, "cannot create '" + path + "': " + std::strerror(errno));
  bool ok = bytes.empty() || std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  if (ok && std::fflush(f) != 0) ok = false;
  if (ok && fsync_file && fsync(fileno(f)) != 0) ok = false;
  if (std::fclose(f) != 0) ok = false;
  if (!ok) fail(ND_ERR_IO, "write failed for '" + path + "'");
}

}  // namespace

void write_report(const std::string& dir, const std::vector<uint64_t>& members,
                  const std::vector<uint64_t>& group_start, const std::vector<uint64_t>& near,
                  const std::vector<uint64_t>& removals, uint64_t total_documents,
                  uint64_t total_records, uint64_t distinct_pairs, bool fsync_files) {
  using ordered_json = nlohmann::ordered_json;
  const uint64_t groups = group_start.empty() ? 0 : group_start.size() - 1;
  std::string lines;
  for (uint64_t g = 0; g < groups; ++g) {
    ordered_json j;
    j["representative"] = members[group_start[g]];
    j["members"] = std::vector<uint64_t>(members.begin() + group_start[g],
                                         members.begin() + group_start[g + 1]);
    lines += j.dump();
    lines += '\n';
  }
  write_file(dir + "/groups.jsonl", lines, fsync_files);  // pipeline.cpp:487

  std::string rem;
  for (uint64_t d : removals) {
    rem += std::to_string(d);
    rem += '\n';
  }
  write_file(dir + "/removal.txt", rem, fsync_files);  // pipeline.cpp:494

  double ratio = total_documents > 0 ? static_cast<double>(near.size()) /
                                           static_cast<double>(total_documents)
                                     : 0.0;
  ordered_json summary;
  summary["total_records"] = total_records;
  summary["total_documents"] = total_documents;
  summary["duplicate_groups"] = groups;
  summary["near_duplicates"] = near.size();
  summary["removals"] = removals.size();
  summary["distinct_pairs"] = distinct_pairs;
  summary["ratio"] = ratio;
  summary["ratio_label"] = std::to_string(near.size()) + " / " + std::to_string(total_documents);
  write_file(dir + "/summary.json", summary.dump(2) + "\n", fsync_files);  // pipeline.cpp:506
}

}  // namespace ndb
