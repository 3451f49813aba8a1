// On-disk artifacts of the staged workflow, byte-identical with the reference:
//   .feds signature files   SignatureFileHeader / Writer / Reader (sigstore.cpp:13-169)
//   .pairs files            write_pair_file / read_pair_file (compare.cpp:88-113)
//   plan_gather             sigstore.cpp:288-329
// Host code (little-endian x86-64: the LE fields are memcpy'd).  Records move
// between the file layout (doc_id u64 | H x u32 | b x u32) and the
// struct-of-arrays layout the kernels use with a few host threads.
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <vector>

#include "host_internal.hpp"

namespace ndb {
namespace {

constexpr char kMagic[4] = {'F', 'E', 'D', 'S'};
constexpr uint32_t kVersion = 1;

template <class T>
void put(std::string& out, T v) {
  out.append(reinterpret_cast<const char*>(&v), sizeof v);
}
template <class T>
T get(const unsigned char* p) {
  T v;
  std::memcpy(&v, p, sizeof v);
  return v;
}

struct File {
  FILE* f = nullptr;
  std::string path;
  File(const std::string& p, const char* mode) : path(p) { f = std::fopen(p.c_str(), mode); }
  ~File() {
    if (f) std::fclose(f);
  }
  // flush + optional fsync + close (write_file_bytes, util.cpp:132-140)
  void finish(bool fsync_file) {
    bool ok = std::fflush(f) == 0;
    if (ok && fsync_file) ok = fsync(fileno(f)) == 0;
    if (std::fclose(f) != 0) ok = false;
    f = nullptr;
    if (!ok) fail(ND_ERR_IO, "write failed for '" + path + "'");
  }
};

unsigned host_threads(uint64_t work) {
  unsigned t = std::max(1u, std::thread::hardware_concurrency());
  return static_cast<unsigned>(std::min<uint64_t>(std::min(t, 32u), std::max<uint64_t>(1, work / 65536)));
}

template <class Fn>
void parallel_ranges(uint64_t n, Fn fn) {
  const unsigned t = host_threads(n);
  if (t <= 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned i = 0; i < t; ++i)
    th.emplace_back([&, i] { fn(n * i / t, n * (i + 1) / t); });
  for (auto& x : th) x.join();
}

}  // namespace

uint64_t feds_record_bytes(const nd_feds_header& h) {
  return 8 + 4ull * h.hash_count + 4ull * h.bands;
}

// SignatureFileHeader::serialize (sigstore.cpp:20-36)
std::string feds_serialize(const nd_feds_header& h) {
  std::string out;
  out.append(kMagic, 4);
  put<uint32_t>(out, kVersion);
  put<uint32_t>(out, h.hash_count);
  put<uint32_t>(out, h.bands);
  put<uint32_t>(out, h.rows);
  put<uint32_t>(out, h.bucket_count);
  put<uint32_t>(out, h.shingle_len);
  put<uint32_t>(out, h.unit);
  put<uint64_t>(out, h.family_seed);
  put<uint64_t>(out, h.scale_num);
  put<uint64_t>(out, h.scale_den);
  put<uint64_t>(out, h.record_count);
  put<uint64_t>(out, h.source_ordinal);
  return out;
}

// SignatureFileHeader::parse (sigstore.cpp:38-72) + the reader's size check
// (sigstore.cpp:138-147).  The ratio is kept as written (Ratio normalises on
// construction in the reference; run_compatible compares normalised values).
nd_feds_header feds_read_header(const std::string& path, uint64_t* file_size) {
  File f(path, "rb");
  if (!f.f) fail(ND_ERR_IO, "cannot open '" + path + "': " + std::strerror(errno));
  unsigned char head[kFedsHeaderBytes];
  const size_t got = std::fread(head, 1, sizeof head, f.f);
  if (got < kFedsHeaderBytes) fail(ND_ERR_IO, "'" + path + "' is shorter than a signature file header");
  if (std::memcmp(head, kMagic, 4) != 0) fail(ND_ERR_IO, "'" + path + "' is not a signature file (bad magic)");
  const uint32_t version = get<uint32_t>(head + 4);
  if (version != kVersion)
    fail(ND_ERR_IO, "'" + path + "' has unsupported signature format version " + std::to_string(version));
  nd_feds_header h{};
  h.hash_count = get<uint32_t>(head + 8);
  h.bands = get<uint32_t>(head + 12);
  h.rows = get<uint32_t>(head + 16);
  h.bucket_count = get<uint32_t>(head + 20);
  h.shingle_len = get<uint32_t>(head + 24);
  h.unit = get<uint32_t>(head + 28);
  if (h.unit > 1) fail(ND_ERR_IO, "'" + path + "' has unknown shingle unit tag");
  h.family_seed = get<uint64_t>(head + 32);
  h.scale_num = get<uint64_t>(head + 40);
  h.scale_den = get<uint64_t>(head + 48);
  if (h.scale_den == 0) fail(ND_ERR_IO, "'" + path + "' has a zero bucket-scale denominator");
  h.record_count = get<uint64_t>(head + 56);
  h.source_ordinal = get<uint64_t>(head + 64);
  if (h.hash_count == 0 || h.bands == 0 || h.rows == 0 || h.bucket_count == 0)
    fail(ND_ERR_IO, "'" + path + "' has zero-valued header parameters");
  struct stat sb;
  if (stat(path.c_str(), &sb) != 0) fail(ND_ERR_IO, "cannot stat '" + path + "': " + std::strerror(errno));
  const uint64_t size = static_cast<uint64_t>(sb.st_size);
  const uint64_t expect = kFedsHeaderBytes + h.record_count * feds_record_bytes(h);
  if (size != expect)
    fail(ND_ERR_IO, "'" + path + "' is corrupt: " + std::to_string(size) + " bytes, header says " +
                        std::to_string(expect));
  if (file_size) *file_size = size;
  return h;
}

namespace {
uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}
// Ratio equality after the reference's normalisation (util.hpp:30-43)
bool same_ratio(uint64_t an, uint64_t ad, uint64_t bn, uint64_t bd) {
  auto norm = [](uint64_t& n, uint64_t& d) {
    uint64_t g = gcd64(n, d);
    if (g) {
      n /= g;
      d /= g;
    }
    if (n == 0) d = 1;
  };
  norm(an, ad);
  norm(bn, bd);
  return an == bn && ad == bd;
}
}  // namespace

// SignatureFileHeader::run_compatible (sigstore.cpp:13-18)
bool feds_run_compatible(const nd_feds_header& a, const nd_feds_header& b) {
  return a.hash_count == b.hash_count && a.bands == b.bands && a.rows == b.rows &&
         a.bucket_count == b.bucket_count && a.shingle_len == b.shingle_len && a.unit == b.unit &&
         a.family_seed == b.family_seed && same_ratio(a.scale_num, a.scale_den, b.scale_num, b.scale_den);
}

// A whole .feds file (SignatureFileWriter, sigstore.cpp:74-130: header, then
// records; record_count is final from the start, the resulting bytes equal
// the reference's header-patched file).
void feds_write(const std::string& path, nd_feds_header h, const uint64_t* doc_ids,
                const uint32_t* sig, const uint32_t* band, uint64_t n, bool fsync_file) {
  h.record_count = n;
  File f(path, "wb");
  if (!f.f) fail(ND_ERR_IO, "cannot create '" + path + "': " + std::strerror(errno));
  const std::string head = feds_serialize(h);
  if (std::fwrite(head.data(), 1, head.size(), f.f) != head.size())
    fail(ND_ERR_IO, "write failed for '" + path + "'");
  const uint64_t H = h.hash_count, B = h.bands, rec = feds_record_bytes(h);
  const uint64_t chunk = std::max<uint64_t>(1, (64ull << 20) / rec);
  std::vector<unsigned char> buf(std::min(n, chunk) * rec);
  for (uint64_t r0 = 0; r0 < n; r0 += chunk) {
    const uint64_t m = std::min(chunk, n - r0);
    parallel_ranges(m, [&](uint64_t a, uint64_t b) {
      for (uint64_t i = a; i < b; ++i) {
        unsigned char* p = buf.data() + i * rec;
        std::memcpy(p, doc_ids + r0 + i, 8);
        std::memcpy(p + 8, sig + (r0 + i) * H, 4 * H);
        std::memcpy(p + 8 + 4 * H, band + (r0 + i) * B, 4 * B);
      }
    });
    if (std::fwrite(buf.data(), 1, m * rec, f.f) != m * rec)
      fail(ND_ERR_IO, "write failed for '" + path + "'");
  }
  f.finish(fsync_file);
}

// All records of one file into struct-of-arrays buffers (SignatureFileReader::
// next, sigstore.cpp:155-175, including the bucket-range corruption check).
void feds_read_records(const std::string& path, const nd_feds_header& h, uint64_t* doc_ids,
                       uint32_t* sig, uint32_t* band) {
  File f(path, "rb");
  if (!f.f) fail(ND_ERR_IO, "cannot open '" + path + "': " + std::strerror(errno));
  if (std::fseek(f.f, static_cast<long>(kFedsHeaderBytes), SEEK_SET) != 0)
    fail(ND_ERR_IO, "'" + path + "' truncated mid-record");
  const uint64_t H = h.hash_count, B = h.bands, rec = feds_record_bytes(h), n = h.record_count;
  const uint64_t chunk = std::max<uint64_t>(1, (64ull << 20) / rec);
  std::vector<unsigned char> buf(std::min(n, chunk) * rec);
  for (uint64_t r0 = 0; r0 < n; r0 += chunk) {
    const uint64_t m = std::min(chunk, n - r0);
    if (std::fread(buf.data(), 1, m * rec, f.f) != m * rec)
      fail(ND_ERR_IO, "'" + path + "' truncated mid-record");
    bool bad = false;
    parallel_ranges(m, [&](uint64_t a, uint64_t b) {
      bool local_bad = false;
      for (uint64_t i = a; i < b; ++i) {
        const unsigned char* p = buf.data() + i * rec;
        if (doc_ids) std::memcpy(doc_ids + r0 + i, p, 8);
        if (sig) std::memcpy(sig + (r0 + i) * H, p + 8, 4 * H);
        uint32_t* bo = band + (r0 + i) * B;
        std::memcpy(bo, p + 8 + 4 * H, 4 * B);
        for (uint64_t j = 0; j < B; ++j) local_bad |= bo[j] >= h.bucket_count;
      }
      if (local_bad) bad = true;  // benign race: only ever set to true
    });
    if (bad) fail(ND_ERR_IO, "'" + path + "' is corrupt: bucket id out of range");
  }
}

// write_pair_file (compare.cpp:88-97): 20-byte LE records lo | hi | match
void pairs_write(const std::string& path, const uint64_t* lo, const uint64_t* hi,
                 const uint32_t* m, uint64_t n, bool fsync_file) {
  File f(path, "wb");
  if (!f.f) fail(ND_ERR_IO, "cannot create '" + path + "': " + std::strerror(errno));
  std::vector<unsigned char> buf(20 * std::min<uint64_t>(n, 1 << 20));
  for (uint64_t r0 = 0; r0 < n; r0 += (1 << 20)) {
    const uint64_t k = std::min<uint64_t>(1 << 20, n - r0);
    for (uint64_t i = 0; i < k; ++i) {
      unsigned char* p = buf.data() + 20 * i;
      std::memcpy(p, lo + r0 + i, 8);
      std::memcpy(p + 8, hi + r0 + i, 8);
      std::memcpy(p + 16, m + r0 + i, 4);
    }
    if (std::fwrite(buf.data(), 1, 20 * k, f.f) != 20 * k)
      fail(ND_ERR_IO, "write failed for '" + path + "'");
  }
  f.finish(fsync_file);
}

// read_pair_file (compare.cpp:99-113); appends
void pairs_read(const std::string& path, std::vector<uint64_t>& lo, std::vector<uint64_t>& hi,
                std::vector<uint32_t>& m) {
  File f(path, "rb");
  if (!f.f) fail(ND_ERR_IO, "cannot open '" + path + "': " + std::strerror(errno));
  struct stat sb;
  if (fstat(fileno(f.f), &sb) != 0) fail(ND_ERR_IO, "read failed for '" + path + "'");
  const uint64_t size = static_cast<uint64_t>(sb.st_size);
  if (size % 20 != 0)
    fail(ND_ERR_IO, "'" + path + "' is corrupt: size is not a multiple of the pair record");
  std::vector<unsigned char> buf(size);
  if (size && std::fread(buf.data(), 1, size, f.f) != size)
    fail(ND_ERR_IO, "read failed for '" + path + "'");
  const uint64_t n = size / 20, base = lo.size();
  lo.resize(base + n);
  hi.resize(base + n);
  m.resize(base + n);
  for (uint64_t i = 0; i < n; ++i) {
    std::memcpy(&lo[base + i], buf.data() + 20 * i, 8);
    std::memcpy(&hi[base + i], buf.data() + 20 * i + 8, 8);
    std::memcpy(&m[base + i], buf.data() + 20 * i + 16, 4);
  }
}

// plan_gather (sigstore.cpp:288-329): C = largest value with
// (total / K) * C * workers <= budget (exact 128-bit), clamped to [1, K];
// passes[w] = number of bucket intervals of width C for workers owning bands.
uint32_t plan_gather(uint64_t total_bytes, uint32_t K, const std::vector<uint32_t>& worker_bands,
                     uint64_t budget, uint32_t override_c, std::vector<uint32_t>& passes) {
  if (K == 0) fail(ND_ERR_CONFIG, "bucket count must be positive");
  if (worker_bands.empty()) fail(ND_ERR_CONFIG, "plan_gather needs at least one worker");
  if (budget == 0) fail(ND_ERR_CONFIG, "memory budget must be positive");
  const uint64_t workers = worker_bands.size();
  uint64_t c;
  if (override_c) {
    c = override_c;
  } else if (total_bytes == 0) {
    c = K;
  } else {
    c = static_cast<uint64_t>(static_cast<unsigned __int128>(budget) * K /
                              (static_cast<unsigned __int128>(total_bytes) * workers));
    if (c < 1)
      fail(ND_ERR_CONFIG, "memory budget " + std::to_string(budget) +
                              " cannot hold even one bucket per worker; raise the budget or the bucket scale");
  }
  if (c > K) c = K;
  passes.assign(workers, 0);
  for (size_t w = 0; w < workers; ++w)
    if (worker_bands[w]) passes[w] = static_cast<uint32_t>((K + c - 1) / c);
  return static_cast<uint32_t>(c);
}

}  // namespace ndb
