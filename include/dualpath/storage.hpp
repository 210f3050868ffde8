// dualpath/storage.hpp — the storage tier: Full Blocks in a file, indexed by
// a trie whose nodes are Full Blocks.
//
// The reference models storage as a byte count only; its
// layout is the paper's: a Full Block is the L Layer Blocks of T tokens
// concatenated, [L][T][b], and the store is a trie in
// which each node is one Full Block of a session prefix.
//
//   FullBlockTrie  — node = Full Block k of a prefix; edge key = the chained
//                    key of that block; node -> record id in the data file.
//   FullBlockFile  — fixed-stride records [L][T][b] (stride rounded up to
//                    4 KiB so O_DIRECT reads land in pinned staging), read with
//                    pread by the executor's IO threads (StorageRead).
//
// Record contents follow the content formula of the procedural store
// (kv_store_fill / oracle/kvref.c): record r holds page r, so a pool loaded
// from the file is byte-identical to one loaded from the procedural store.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <unordered_map>
#include <vector>

#include "dualpath/kv_abi.h"

namespace dualpath {

// 64-bit FNV-1a of a session id: the root key of its chain.
std::uint64_t session_key(const std::string& id);
// Chained key of the first n Full Blocks of a session: key_k depends on every
// block before it (a prefix key, as a content-addressed KV store has).
std::vector<std::uint64_t> session_chain(const std::string& id, std::int64_t n_blocks);

class FullBlockTrie {
 public:
  // Adds the path `chain` (one key per Full Block, in order).  A node created
  // here gets the record id records[depth]; existing nodes keep theirs.
  // Returns the record id of every node on the path.
  std::vector<std::int64_t> insert(std::span<const std::uint64_t> chain,
                                   std::span<const std::int64_t> records);
  // Record ids of the longest prefix of `chain` present in the trie.
  std::vector<std::int64_t> match(std::span<const std::uint64_t> chain) const;
  std::int64_t nodes() const { return static_cast<std::int64_t>(nodes_.size()); }

  // Binary index file: magic, node count, then {parent, key, record} per node.
  void save(const std::string& path) const;
  static FullBlockTrie load(const std::string& path);

 private:
  struct Node {
    std::int64_t parent;
    std::uint64_t key;
    std::int64_t record;
  };
  struct EdgeHash {
    std::size_t operator()(const std::pair<std::int64_t, std::uint64_t>& e) const {
      return std::hash<std::uint64_t>()(e.second ^ (static_cast<std::uint64_t>(e.first) * 0x9E3779B97F4A7C15ull));
    }
  };
  std::vector<Node> nodes_;
  std::unordered_map<std::pair<std::int64_t, std::uint64_t>, std::int64_t, EdgeHash> child_;
};

// Host restatement of the store's content formula: Full Block `page`.
void fill_full_block(const dp_kv_geom& g, std::uint64_t seed, std::int64_t page, void* dst);

class FullBlockFile {
 public:
  // Opens (create: creates / truncates) a file of n_records records.
  // direct: read with O_DIRECT when the file system allows it.
  FullBlockFile(const std::string& path, const dp_kv_geom& g, std::int64_t n_records, bool create,
                bool direct);
  ~FullBlockFile();
  FullBlockFile(const FullBlockFile&) = delete;
  FullBlockFile& operator=(const FullBlockFile&) = delete;

  std::int64_t records() const { return n_records_; }
  std::int64_t record_bytes() const { return record_bytes_; }
  std::int64_t stride() const { return stride_; }
  bool direct() const { return fd_direct_ >= 0; }

  // Writes records [0, n) with the content formula (threads in parallel).
  void populate(std::uint64_t seed, int threads);
  void write(std::int64_t record, const void* src);
  // Writes bytes [offset, offset + n) of a record (buffered).
  void write_bytes(std::int64_t record, std::int64_t offset, std::int64_t n, const void* src);
  // Reads one record into dst (O_DIRECT when dst is 4 KiB aligned and the
  // file was opened direct; buffered otherwise).  Throws on a short read.
  void read(std::int64_t record, void* dst) const;
  // Reads records [record, record + n) into n consecutive Full Blocks at dst:
  // one pread when records are packed (stride == record bytes), else n.
  void read_run(std::int64_t record, std::int64_t n, void* dst) const;

 private:
  std::string path_;
  dp_kv_geom geom_{};
  std::int64_t n_records_ = 0;
  std::int64_t record_bytes_ = 0;
  std::int64_t stride_ = 0;
  int fd_ = -1;
  int fd_direct_ = -1;
};

}  // namespace dualpath
