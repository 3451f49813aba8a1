/* neardup_b200 -- C-ABI of the B200-native MinHash-LSH dedup hot path.
 *
 * The reference (neardup, /root/reference/proj) has no FFI: its boundary is the
 * C++ library API in include/neardup/*.hpp called by src/pipeline.cpp.  Each
 * entry point below replaces one of those calls (cited as file:line under
 * /root/reference/proj); include/neardup_b200.hpp re-exposes them with the
 * reference's C++ names and types.  Plain pointers and sizes only; no
 * allocation crosses the ABI except through the documented two-phase
 * fetch calls.  Status codes mirror the reference's exception taxonomy
 * (util.hpp:13-26 -> tools/main.cpp:18-21 exit codes) plus a device code.
 */
#ifndef NEARDUP_B200_H
#define NEARDUP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define ND_OK 0
#define ND_ERR_INTERNAL 1   /* unexpected failure (bug) */
#define ND_ERR_CONFIG 2     /* ConfigError        util.hpp:13 */
#define ND_ERR_IO 3         /* IoError            util.hpp:18 */
#define ND_ERR_PREREQ 4     /* PrerequisiteError  util.hpp:23 */
#define ND_ERR_DEVICE 5     /* CUDA / NCCL failure (new) */
#define ND_ERR_SHORT 6      /* ShortDocumentError minhash.hpp:63 */

/* HashFunctionParams (minhash.hpp:17-25), byte-identical layout (24 bytes). */
typedef struct nd_hash_fn {
  uint32_t modulus;      /* prime p (derive_family: [2^21, 2^23); GPU path: < 2^31) */
  uint32_t base;         /* prime q (derive_family: (256, 2^16)) */
  uint32_t base_inverse; /* q^-1 mod p */
  uint32_t base_power;   /* q^(L-1) mod p */
  uint64_t reduce_factor;/* floor(2^64 / p) */
} nd_hash_fn;

/* Artifact-shaping run parameters (RunConfig, pipeline.hpp:21-36). */
typedef struct nd_params {
  uint32_t hash_count;      /* H = bands * rows */
  uint32_t bands;           /* b */
  uint32_t rows;            /* r */
  uint32_t shingle_len;     /* L */
  uint32_t unit;            /* 0 = byte (ShingleUnit::kByte); 1 = codepoint (kCodepoint) */
  uint32_t bucket_count;    /* K; 0 = choose_bucket_count(n, bucket_scale) */
  uint64_t threshold_num;   /* SimilarityThreshold (compare.hpp:28-37) */
  uint64_t threshold_den;
  uint64_t scale_num;       /* bucket_scale Ratio (lsh.hpp:18) */
  uint64_t scale_den;
  uint64_t seed;            /* family seed (pipeline.hpp:35) */
} nd_params;

typedef struct nd_ctx nd_ctx;

/* ---- host-only helpers (no device needed) -------------------------------- */
const char* nd_version(void);
/* number of neardup_b200 kernel launches issued by this process so far */
uint64_t nd_launch_count(void);
/* last error message of the calling thread (ctx-free calls) */
const char* nd_last_error_global(void);
/* derive_family (minhash.hpp:42, minhash.cpp:71-105); out holds H entries */
int nd_derive_family(uint64_t seed, uint32_t hash_count, uint32_t shingle_len, uint32_t unit,
                     nd_hash_fn* out);
/* scalar primitives of minhash.hpp (host; minhash.cpp:10-50, :111-131):
 * mod_pow (ND_ERR_CONFIG for a zero modulus), Miller-Rabin is_prime_u32,
 * hash_window_direct (Horner, ND_ERR_CONFIG for an empty window) and the
 * Eq. 5 roll_next -- the per-window arithmetic K1 replaces */
int nd_mod_pow(uint64_t base, uint64_t exp, uint64_t mod, uint64_t* out);
int nd_is_prime_u32(uint32_t n);
int nd_hash_window_direct(const uint32_t* window, uint32_t len, const nd_hash_fn* fn,
                          uint32_t* out);
uint32_t nd_roll_next(uint32_t state, uint32_t outgoing, uint32_t incoming, const nd_hash_fn* fn);
/* choose_bucket_count (lsh.hpp:33, lsh.cpp:26-40) */
int nd_choose_bucket_count(uint64_t doc_count, uint64_t scale_num, uint64_t scale_den,
                           uint32_t* bucket_count_out);
/* SimilarityThreshold::min_matches (compare.hpp:35, compare.cpp:17-22) */
uint32_t nd_min_matches(uint32_t hash_count, uint64_t num, uint64_t den);
/* band_partition (lsh.hpp:53, lsh.cpp:62-72): ranges[2*w], ranges[2*w+1] */
int nd_band_partition(uint32_t bands, uint32_t workers, uint32_t* ranges);
/* cell owner map for G shards: owner(cell) = floor(cell * G / (bands*K)); the
 * generalisation of band_partition to cell ranges. first_cell has
 * G+1 entries. */
int nd_cell_partition(uint32_t bands, uint32_t bucket_count, uint32_t shards,
                      uint64_t* first_cell);

/* Seeded synthetic corpus in the reference generator's shape
 * (synthetic.cpp:39-110).  mode 0 reproduces generate_synthetic bit for bit
 * (single thread); mode 1 is the multi-threaded streaming variant for large
 * corpora (same alphabet, length law, groups, edit law; different RNG
 * stream).  len_law 0 = uniform [len_min, len_max]; 1 = lognormal with
 * median len_min, sigma_milli/1000, clipped to [200, len_max].
 * Two-phase: call with bytes == NULL to learn nbytes, then again to fill. */
typedef struct nd_synth_spec {
  uint64_t doc_count, group_count;
  uint32_t group_size_min, group_size_max;
  uint64_t edit_num, edit_den;
  uint32_t len_min, len_max;
  uint64_t seed;
  uint32_t mode, len_law, sigma_milli, threads;
} nd_synth_spec;
int nd_synth_generate(const nd_synth_spec* spec, uint8_t* bytes, uint64_t* offsets,
                      uint64_t* nbytes_out);
/* mode-1 corpus text generated directly in device memory (identical bytes to
 * nd_synth_generate); d_offsets = the offsets nd_synth_generate(spec, NULL,
 * offsets, &n) returned, already copied to the device.  Synchronous. */
int nd_synth_text_device(nd_ctx* ctx, const nd_synth_spec* spec, const uint64_t* d_offsets,
                         uint8_t* d_bytes);

/* ---- device context ----------------------------------------------------- */
int nd_ctx_create(int device, nd_ctx** out);
/* One context over several devices (the reference's in-process
 * parallel compare, pipeline.cpp:387-420, band_partition lsh.cpp:62-72):
 * one host thread per shard, peer access enabled between distinct devices.
 * nd_signatures and nd_dedup shard the batch by contiguous document ranges;
 * nd_dedup exchanges (cell, row) records all-to-all over NVLink peer copies,
 * every owner compares its cells reading signature rows in place from the
 * owning GPU, and the pairs meet on the first device for the components.
 * Outputs are identical for any device list; a device may repeat (several
 * shards on one GPU).  The fetch / report calls work on the group context;
 * other entry points run on the first device. */
int nd_ctx_create_multi(const int* devices, int ndev, nd_ctx** out);
int nd_ctx_shard_count(const nd_ctx* ctx);
void nd_ctx_destroy(nd_ctx* ctx);
const char* nd_last_error(const nd_ctx* ctx);
/* stream all device work of this ctx is ordered on (cudaStream_t; NULL = own) */
int nd_ctx_set_stream(nd_ctx* ctx, void* cuda_stream);
/* Uploads the family (derive_family's output, or a hand-built one) for the
 * signature kernels.  ND_ERR_CONFIG unless every function meets the
 * reference's own preconditions: modulus above the largest unit
 * (minhash.cpp:107-109), modulus < 2^31, base_inverse / base_power /
 * reduce_factor as derive_family computes them (minhash.cpp:99-101).
 * derive_family's domain (2^21 <= p < 2^23, q < 2^16) runs the FP32-quotient
 * kernel; any other accepted family runs the reference's 64-bit Barrett
 * reduction (exact, slower). */
int nd_family_upload(nd_ctx* ctx, const nd_hash_fn* fns, uint32_t hash_count,
                     uint32_t shingle_len, uint32_t unit);
/* Which signature kernel the uploaded family runs: "k1j" (family-specialised,
 * compiled by NVRTC at upload), "k1" (per-lane register constants), "k1w"
 * (codepoint units), "k1j+k1w" / "k1+k1w" (codepoint units: documents whose
 * code points are all < 256 on the byte kernel, the others on K1w) or "k1x"
 * (exact 64-bit Barrett); when K1j was eligible but could not be compiled the
 * reason follows after ": ". */
const char* nd_k1_kernel(nd_ctx* ctx);
/* How the last nd_dedup / nd_dedup_device compared: "global" (one block join
 * over all rows, the cells counted for the reference's counters; the
 * in-memory default, on a device group each block joined by one shard),
 * "cells" (the per-cell joins: out-of-core intervals, thresholds with more
 * than 64 blocks, ND_K3=cells) or "" (no valid dedup). */
const char* nd_dedup_compare_kind(nd_ctx* ctx);
/* The CUDA source K1j compiles for a family (no device needed): writes up to
 * cap bytes (NUL-terminated) into out and returns the full length, or -1
 * when the family is outside K1j's domain. */
int64_t nd_k1j_source(const nd_hash_fn* fns, uint32_t hash_count, uint32_t shingle_len, char* out,
                      uint64_t cap);
/* The same for K1j over 16-bit units (unit_bytes = 2: codepoint documents
 * whose code points are all < 2^16, the fq arithmetic; unit_bytes = 1 is
 * nd_k1j_source). */
int64_t nd_k1j_source_units(const nd_hash_fn* fns, uint32_t hash_count, uint32_t shingle_len,
                            uint32_t unit_bytes, char* out, uint64_t cap);
/* K1j's dn plan for a family (no device needed): per function one row of 12
 * u32 {pass, class, g, w, function, q, QLn, Kb multiplier, p, A bits, B bits,
 * M bits} (csrc/k1_jit.cpp, the denormal-state arithmetic), written up to
 * cap_rows rows; returns the row count (= hash_count) or -1 when the family
 * runs another arithmetic (outside the fq domain, ND_K1J_ARITH=fq). */
int64_t nd_k1j_plan(const nd_hash_fn* fns, uint32_t hash_count, uint32_t shingle_len, uint32_t* out,
                    uint64_t cap_rows);

/* signature_of_document over a packed batch + band_bucket_ids
 * (minhash.hpp:71-78, lsh.hpp:38-40; caller pipeline.cpp:214-218).
 * bytes[offsets[i] .. offsets[i+1]) is document i (NFC UTF-8); its units are
 * the bytes, or the decoded scalar values when the family was uploaded with
 * unit 1 (text_units, text.cpp:115-122; decoded on the GPU).
 * sig_out: n*H u32 row-major; band_out: n*bands u32 (NULL to skip), ids mod K
 * (K == 0 -> raw u32 band row sums, K-independent).  Every document must
 * yield a full window (else ND_ERR_SHORT, nothing written).
 * Host pointers; copies in and out are pipelined inside; synchronous. */
int nd_signatures(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                  uint32_t bands, uint32_t rows, uint32_t bucket_count, uint32_t* sig_out,
                  uint32_t* band_out);
/* Host text in, device outputs: the same pipelined H2D + K1 as nd_signatures
 * but d_sig / d_band stay in HBM (input of the dedup stages).  Synchronous. */
int nd_signatures_h2d(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                      uint32_t bands, uint32_t rows, uint32_t bucket_count, uint32_t* d_sig,
                      uint32_t* d_band);
/* Same on device pointers, asynchronous on the ctx stream. */
int nd_signatures_device(nd_ctx* ctx, const uint8_t* d_bytes, const uint64_t* d_offsets,
                         uint64_t n, uint32_t bands, uint32_t rows, uint32_t bucket_count,
                         uint32_t* d_sig, uint32_t* d_band);

/* text_units (text.hpp:32, text.cpp:101-122) over a packed batch, on the GPU:
 * unit_offsets[n+1] (prefix sums of per-document unit counts; the counts are
 * codepoint_count, text.cpp:88-99) and, when units_out is not NULL, the units
 * (bytes widened, or scalar values with U+FFFD per ill-formed subpart).
 * Call once with units_out = NULL to size the buffer.  Synchronous. */
int nd_text_units(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                  uint32_t unit, uint64_t* unit_offsets, uint32_t* units_out);

/* band_bucket_ids (lsh.hpp:38-40, lsh.cpp:42-60) over host signature rows
 * sigs[n*H] -> band ids[n*bands] (K == 0: raw u32 row sums). */
int nd_band_keys(nd_ctx* ctx, const uint32_t* sigs, uint64_t n, uint32_t hash_count,
                 uint32_t bands, uint32_t rows, uint32_t bucket_count, uint32_t* band_out);

/* compare_pass (compare.hpp:52, compare.cpp:69-86) over cells given as CSR
 * row lists into a host signature matrix sigs[nrows*H]; rows inside a cell
 * ascend.  Result: sorted distinct (lo, hi) row pairs with match counts,
 * fetched with nd_pairs_fetch. */
int nd_compare_cells(nd_ctx* ctx, const uint32_t* sigs, uint64_t nrows, uint32_t hash_count,
                     const uint64_t* cell_offsets, const uint32_t* cell_rows, uint64_t ncells,
                     uint64_t threshold_num, uint64_t threshold_den, uint64_t* npairs_out);
int nd_pairs_fetch(nd_ctx* ctx, uint32_t* lo, uint32_t* hi, uint32_t* match_count);

/* union_pairs + components (dedup_graph.hpp:34-43) over row-index pairs;
 * groups fetched with nd_groups_fetch. */
int nd_union(nd_ctx* ctx, const uint32_t* lo, const uint32_t* hi, uint64_t npairs,
             uint32_t nnodes, uint64_t* nmembers_out, uint64_t* ngroups_out);
/* members in output order (groups by representative, members ascending);
 * group_start[ngroups+1] offsets into members. */
int nd_groups_fetch(nd_ctx* ctx, uint32_t* members, uint64_t* group_start);

/* In-memory run_dedup (pipeline.hpp:100, pipeline.cpp:510-532): signatures
 * -> band keys -> cell grouping -> compare -> distinct pairs -> components.
 * doc_ids (NULL = 0..n-1) must ascend.  Stats then fetch. */
typedef struct nd_dedup_stats {
  uint64_t documents;        /* total_surviving */
  uint32_t bucket_count;     /* K used */
  uint64_t nonsingleton_cells;
  uint64_t candidate_pairs;  /* sum n(n-1)/2 over cells (pipeline.cpp:406-411) */
  uint64_t emitted_pairs;    /* accepted before cross-band dedup */
  uint64_t distinct_pairs;
  uint64_t duplicate_groups;
  uint64_t near_duplicates;
  uint64_t removals;
  double seconds[6];         /* device time: sig (K1), cells (K2), compare (K3),
                                distinct pairs (K4a sort + unique), cc (K4), d2h */
  uint64_t cell_records;     /* sum of n over the non-singleton cells (K3's rows) */
  uint32_t intervals;        /* bucket intervals (1 = everything resident in HBM) */
} nd_dedup_stats;
int nd_dedup(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, const uint64_t* doc_ids,
             uint64_t n, const nd_params* params, nd_dedup_stats* stats);
/* Same with the packed batch already in device memory. */
int nd_dedup_device(nd_ctx* ctx, const uint8_t* d_bytes, const uint64_t* d_offsets,
                    const uint64_t* doc_ids, uint64_t n, const nd_params* params,
                    nd_dedup_stats* stats);
/* The same dedup from signature rows already computed (e.g. read from .feds
 * files with nd_feds_read): sig n*hash_count u32, band n*bands u32 host
 * arrays, every band id below the bucket count (params->bucket_count, or
 * choose_bucket_count(n)); compare + distinct pairs + components in HBM
 * (run_compare_stage + run_union_stage, pipeline.cpp:347-476, in memory). */
int nd_dedup_signatures(nd_ctx* ctx, const uint32_t* sig, const uint32_t* band,
                        const uint64_t* doc_ids, uint64_t n, const nd_params* params,
                        nd_dedup_stats* stats);
/* distinct pairs (doc ids, sorted by (lo, hi)) of the last dedup */
int nd_dedup_fetch_pairs(nd_ctx* ctx, uint64_t* lo, uint64_t* hi, uint32_t* match_count);
/* signatures (n*H u32) and band ids (n*bands u32) the last dedup computed,
 * rows in input order (either output may be NULL) */
int nd_dedup_fetch_signatures(nd_ctx* ctx, uint32_t* sig, uint32_t* band);
/* groups of the last dedup as doc ids: members in output order,
 * group_start[ngroups+1]; representative = members[group_start[g]] */
int nd_dedup_fetch_groups(nd_ctx* ctx, uint64_t* members, uint64_t* group_start);
/* Reference-identical report bytes (groups.jsonl, removal.txt, summary.json
 * as written by pipeline.cpp:479-506) for the last dedup, into dir. */
int nd_dedup_write_report(nd_ctx* ctx, const char* dir, uint64_t total_records);
/* Same; fsync_files != 0 fsyncs each file before closing it, as the
 * reference's write_file_bytes does under --fsync (util.cpp:132-140,
 * pipeline.cpp:487-506). */
int nd_dedup_write_report_ex(nd_ctx* ctx, const char* dir, uint64_t total_records,
                             int fsync_files);

/* ---- host document loader (corpus.cpp / text.cpp), multi-threaded C++ ------
 * One JSONL file per call: lines split as for_each_raw_document
 * (corpus.cpp:56-82), parsed by parse_jsonl_line's parser (nlohmann::json,
 * corpus.cpp:31-54), NFC-normalised (text.cpp:70-86; UAX #15 tables from the
 * UCD), code points counted and filtered by min_chars / can_shingle
 * (corpus.cpp:93-141).  Reject reason codes: 1 invalid_json, 2 not_an_object,
 * 3 missing_text_field, 4 text_field_not_string, 5 below_min_chars,
 * 6 too_short_to_shingle.  Errors: nd_ingest_last_error(). */
typedef struct nd_jsonl nd_jsonl;
const char* nd_ingest_last_error(void);
int nd_jsonl_load(const char* path, const char* text_field, uint64_t min_chars,
                  uint32_t shingle_len, uint32_t unit, uint32_t threads, int keep_text,
                  nd_jsonl** out);
void nd_jsonl_counts(const nd_jsonl* f, uint64_t* records, uint64_t* surviving,
                     uint64_t* text_bytes, uint64_t* rejects);
/* rejects in line order: 1-based line numbers and reason codes */
int nd_jsonl_rejects(const nd_jsonl* f, uint64_t* lines, uint32_t* reasons);
/* the surviving documents, doc_id = record_offset + record ordinal
 * (preprocess, corpus.cpp:93-101); bytes/offsets[n+1] need keep_text */
int nd_jsonl_documents(const nd_jsonl* f, uint64_t record_offset, uint8_t* bytes,
                       uint64_t* offsets, uint64_t* doc_ids, uint64_t* char_counts);
void nd_jsonl_free(nd_jsonl* f);
/* nfc_normalize (text.cpp:70-86): *out_len always set; copied when cap suffices */
int nd_nfc_normalize(const uint8_t* in, uint64_t len, uint8_t* out, uint64_t cap,
                     uint64_t* out_len);
/* codepoint_count (text.cpp:88-99) */
uint64_t nd_codepoint_count(const uint8_t* s, uint64_t len);
/* parse_jsonl_line (corpus.cpp:31-54): *reason 0 = ok (text copied when cap suffices) */
int nd_parse_jsonl_line(const char* line, uint64_t len, const char* text_field, uint32_t* reason,
                        uint8_t* text_out, uint64_t cap, uint64_t* text_len);
/* same with the parser chosen: 0 fast scanner then nlohmann (the default),
 * 1 nlohmann only, 2 fast scanner only (*reason 255 = undecided) */
int nd_parse_jsonl_line_mode(const char* line, uint64_t len, const char* text_field, int mode,
                             uint32_t* reason, uint8_t* text_out, uint64_t cap, uint64_t* text_len);

/* ---- staged workflow on disk: hash -> gather-compare -> union ---------------
 * The reference persists every stage (pipeline.hpp:62-96): one .feds signature
 * file per input file, one .pairs file per (worker, gather pass), then the
 * report.  These entry points produce and consume the same bytes, so stages
 * can be mixed with the reference's (e.g. its union stage on our pair files). */
typedef struct nd_feds_header { /* SignatureFileHeader (sigstore.hpp:24-42) */
  uint32_t hash_count, bands, rows, bucket_count, shingle_len, unit;
  uint64_t family_seed, scale_num, scale_den, record_count, source_ordinal;
} nd_feds_header;
/* SignatureFileWriter (sigstore.cpp:74-130) for n records; record_count is
 * set to n.  sig: n*H u32 row-major, band: n*bands u32. */
int nd_feds_write(const char* path, const nd_feds_header* header, const uint64_t* doc_ids,
                  const uint32_t* sig, const uint32_t* band, uint64_t n, int fsync_file);
/* SignatureFileHeader::parse + the reader's size check (sigstore.cpp:38-72, :132-150) */
int nd_feds_read_header(const char* path, nd_feds_header* out);
/* SignatureFileReader::next over the whole file (sigstore.cpp:155-175);
 * any output may be NULL except band (checked against bucket_count). */
int nd_feds_read(const char* path, uint64_t* doc_ids, uint32_t* sig, uint32_t* band);
/* write_pair_file / read_pair_file (compare.cpp:88-113); read: call with
 * NULL outputs to get *n, then again with buffers of *n entries. */
int nd_pairs_write(const char* path, const uint64_t* lo, const uint64_t* hi, const uint32_t* match,
                   uint64_t n, int fsync_file);
int nd_pairs_read(const char* path, uint64_t* lo, uint64_t* hi, uint32_t* match, uint64_t* n);
/* plan_gather (sigstore.cpp:288-329) with band_partition's worker ranges
 * (lsh.cpp:62-72): buckets per pass C and passes[w] per worker (0 for a
 * worker without bands).  override_c: 0 = none. */
int nd_plan_gather(uint64_t total_signature_bytes, uint32_t bucket_count, uint32_t bands,
                   uint32_t workers, uint64_t memory_budget, uint32_t override_c,
                   uint32_t* c_out, uint32_t* passes_out);
/* hash_one_file (pipeline.cpp:171-240) for one input file: K1 on the GPU over
 * its packed surviving documents (doc_ids ascending), written to path as a
 * .feds file.  The family is derived from the header (seed, H, L, unit). */
int nd_hash_file(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets,
                 const uint64_t* doc_ids, uint64_t n, const nd_feds_header* header,
                 const char* path, int fsync_file);
typedef struct nd_compare_stage_stats { /* CompareStageOutput (pipeline.hpp:74-81) */
  uint32_t buckets_per_pass, pass_count;
  uint64_t candidate_pairs, emitted_pairs, gather_peak_bytes;
  uint64_t records;          /* signature records read */
  uint64_t distinct_pairs;   /* summed over bucket intervals */
  double seconds[3];         /* read, GPU compare (all intervals), pair files */
  uint32_t intervals;        /* bucket intervals the cells went to the GPU in */
} nd_compare_stage_stats;
/* HBM the compare stage may fill with one bucket interval's signatures and
 * cell records (0 = 70 % of the free device memory).  Corpora above it are
 * compared in several intervals (out-of-core), each a union of whole gather
 * passes, with identical output files. */
int nd_set_hbm_budget(nd_ctx* ctx, uint64_t bytes);
/* run_compare_stage (pipeline.cpp:347-432) minus its JSON: every .feds file
 * (source order) is loaded into HBM once; the cells of all passes are
 * compared on the GPU and each pass's sorted distinct pairs are written to
 * pairs_dir/w<w>_p<p>.pairs (an empty file for a pass without pairs), the
 * files compare_pass + write_pair_file would produce.  expected: the run's
 * header (record_count / source_ordinal ignored).  gather_peak_bytes is the
 * resident bytes scan_gather would hold: exact for one worker, the
 * passes-in-lockstep sum for several. */
int nd_compare_stage(nd_ctx* ctx, const char* const* feds_paths, uint32_t nfiles,
                     const nd_feds_header* expected, uint64_t total_signature_bytes,
                     uint32_t workers, uint64_t memory_budget, uint32_t buckets_per_pass,
                     uint64_t threshold_num, uint64_t threshold_den, const char* pairs_dir,
                     int fsync_files, nd_compare_stage_stats* stats);
/* run_union_stage (pipeline.cpp:434-508) minus its JSON checks: reads the
 * pair files, distinct pairs + components on the GPU, writes groups.jsonl,
 * removal.txt and summary.json into workspace.  Result also fetchable with
 * nd_dedup_fetch_*. */
int nd_union_stage(nd_ctx* ctx, const char* const* pair_paths, uint32_t nfiles,
                   uint64_t total_surviving, uint64_t total_records, const char* workspace,
                   int fsync_files, nd_dedup_stats* stats);

/* ---- stage entry points for the multi-GPU dedup (device pointers, async on
 * the ctx stream unless noted).  See DESIGN.md section 7. -------------------- */
/* (cell = band*K + bucket, doc_base + row) records of n documents' band ids,
 * stably sorted by cell (scan_gather's grouping, sigstore.cpp:228-286);
 * d_keys / d_vals receive n*bands entries each. */
int nd_stage_cell_records(nd_ctx* ctx, const uint32_t* d_band, uint64_t n, uint32_t bands,
                          uint32_t bucket_count, uint32_t doc_base, uint32_t* d_keys,
                          uint32_t* d_vals);
/* The same records packed for one all-to-all: d_rec[i] = cell << 32 | row,
 * sorted by cell, and owner_split[world + 1] (host) = where each owner's run
 * starts (owner of a cell = nd_cell_partition(bands, K, world)).
 * Synchronous (the splits are read back). */
int nd_stage_records_packed(nd_ctx* ctx, const uint32_t* d_band, uint64_t n, uint32_t bands,
                            uint32_t bucket_count, uint32_t doc_base, uint32_t world,
                            uint64_t* d_rec, uint64_t* owner_split);
/* nd_stage_compare_peer over m packed records (arrival order = rank order). */
int nd_stage_compare_peer_packed(nd_ctx* ctx, const uint64_t* d_rec, uint64_t m,
                                 uint64_t key_limit, uint64_t threshold_num,
                                 uint64_t threshold_den, uint64_t* npairs_out,
                                 uint64_t* candidate_pairs_out);
/* compare_pass over the cells of m (cell, row) records (any order; stable by
 * arrival) against signature rows d_sig[nrows*H]; keeps the sorted distinct
 * pairs in the ctx; synchronous; *npairs_out = their count. */
int nd_stage_compare(nd_ctx* ctx, const uint32_t* d_sig, uint64_t nrows, uint32_t hash_count,
                     const uint32_t* d_keys, const uint32_t* d_vals, uint64_t m,
                     uint64_t key_limit, uint64_t threshold_num, uint64_t threshold_den,
                     uint64_t* npairs_out, uint64_t* candidate_pairs_out);
/* ---- compare over peer memory (replaces the all-gather of signature rows) ---
 * Each rank exports its rows (copied into a ctx-owned allocation) as a CUDA
 * IPC handle; after the handles are all-gathered, nd_peer_open maps the other
 * ranks' rows (NVLink peer memory) and nd_stage_compare_peer runs
 * nd_stage_compare with global row g read from the rank r where
 * row_base[r] <= g < row_base[r+1].  Keep the exported rows alive (no
 * nd_peer_close) until every rank has finished comparing. */
#define ND_IPC_HANDLE_BYTES 64
int nd_peer_export(nd_ctx* ctx, const uint32_t* d_sig, uint64_t rows, uint32_t hash_count,
                   uint8_t* handle_out);
int nd_peer_open(nd_ctx* ctx, const uint8_t* handles, const uint64_t* row_base, uint32_t world,
                 uint32_t self);
int nd_stage_compare_peer(nd_ctx* ctx, const uint32_t* d_keys, const uint32_t* d_vals,
                          uint64_t m, uint64_t key_limit, uint64_t threshold_num,
                          uint64_t threshold_den, uint64_t* npairs_out, uint64_t* candidate_pairs_out);
int nd_peer_close(nd_ctx* ctx);
/* K3g over peer memory (the global block join, one process per GPU): each
 * rank exports, in one IPC allocation, its signature rows, its band ids and
 * the block fingerprints of its rows for the threshold; after nd_peer_open,
 * nd_stage_gjoin_peer joins the blocks k = self (mod world) over ALL ranks'
 * rows (global row ids) -- every accepted pair of the batch is found by
 * exactly one rank -- leaving distinct pairs for nd_stage_pairs_copy and the
 * rank's share of the emitted-pairs counter.  nd_stage_cell_hist writes this
 * rank's cell histogram (bands*K u32, d_cnt) for an all-reduce: the
 * reference's counters (pipeline.cpp:406-411) come from the summed one. */
int nd_peer_export_gjoin(nd_ctx* ctx, const uint32_t* d_sig, const uint32_t* d_band, uint64_t rows,
                         uint32_t hash_count, uint32_t bands, uint64_t threshold_num,
                         uint64_t threshold_den, uint8_t* handle_out);
int nd_stage_gjoin_peer(nd_ctx* ctx, uint32_t self, uint64_t* npairs_out, uint64_t* emitted_out);
int nd_stage_cell_hist(nd_ctx* ctx, const uint32_t* d_band, uint64_t n, uint32_t bands, uint32_t K,
                       uint32_t* d_cnt);
/* copies the pairs of the last nd_stage_compare into device buffers */
int nd_stage_pairs_copy(nd_ctx* ctx, uint32_t* d_lo, uint32_t* d_hi, uint32_t* d_match);
/* union stage over gathered pairs (rows < nnodes, repeats allowed): distinct
 * pairs + components become the ctx's dedup result (nd_dedup_fetch_* and
 * nd_dedup_write_report apply; doc ids = rows).  Synchronous. */
int nd_stage_union(nd_ctx* ctx, const uint32_t* d_lo, const uint32_t* d_hi,
                   const uint32_t* d_match, uint64_t npairs, uint64_t nnodes,
                   nd_dedup_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* NEARDUP_B200_H */
