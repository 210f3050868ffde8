// The storage tier (see dualpath/storage.hpp).
#include "dualpath/storage.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <thread>

namespace dualpath {

namespace {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr std::uint64_t kSeedMul = 0xD1B54A32D192ED03ull;
constexpr std::int64_t kAlign = 4096;
constexpr std::uint64_t kTrieMagic = 0x3145495254424644ull;  // "DFBTRIE1"

std::uint64_t splitmix64(std::uint64_t x) {
  std::uint64_t z = x + kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

[[noreturn]] void io_error(const std::string& what, const std::string& path) {
  throw std::runtime_error(what + " " + path + ": " + std::strerror(errno));
}

}  // namespace

std::uint64_t session_key(const std::string& id) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : id) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

std::vector<std::uint64_t> session_chain(const std::string& id, std::int64_t n_blocks) {
  std::vector<std::uint64_t> chain;
  chain.reserve(static_cast<std::size_t>(std::max<std::int64_t>(0, n_blocks)));
  std::uint64_t key = session_key(id);
  for (std::int64_t k = 0; k < n_blocks; ++k) {
    key = splitmix64(key ^ splitmix64(static_cast<std::uint64_t>(k) + kGolden));
    chain.push_back(key);
  }
  return chain;
}

std::vector<std::int64_t> FullBlockTrie::insert(std::span<const std::uint64_t> chain,
                                                std::span<const std::int64_t> records) {
  if (records.size() < chain.size()) throw std::invalid_argument("FullBlockTrie::insert: too few records");
  std::vector<std::int64_t> out;
  out.reserve(chain.size());
  std::int64_t at = -1;  // the root
  for (std::size_t d = 0; d < chain.size(); ++d) {
    const auto edge = std::make_pair(at, chain[d]);
    auto it = child_.find(edge);
    if (it == child_.end()) {
      nodes_.push_back({at, chain[d], records[d]});
      it = child_.emplace(edge, static_cast<std::int64_t>(nodes_.size() - 1)).first;
    }
    at = it->second;
    out.push_back(nodes_[at].record);
  }
  return out;
}

std::vector<std::int64_t> FullBlockTrie::match(std::span<const std::uint64_t> chain) const {
  std::vector<std::int64_t> out;
  std::int64_t at = -1;
  for (std::uint64_t key : chain) {
    const auto it = child_.find(std::make_pair(at, key));
    if (it == child_.end()) break;
    at = it->second;
    out.push_back(nodes_[at].record);
  }
  return out;
}

void FullBlockTrie::save(const std::string& path) const {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) io_error("cannot write trie index", path);
  const std::uint64_t n = nodes_.size();
  f.write(reinterpret_cast<const char*>(&kTrieMagic), 8);
  f.write(reinterpret_cast<const char*>(&n), 8);
  for (const Node& node : nodes_) {
    f.write(reinterpret_cast<const char*>(&node.parent), 8);
    f.write(reinterpret_cast<const char*>(&node.key), 8);
    f.write(reinterpret_cast<const char*>(&node.record), 8);
  }
  if (!f) io_error("short write of trie index", path);
}

FullBlockTrie FullBlockTrie::load(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) io_error("cannot read trie index", path);
  std::uint64_t magic = 0, n = 0;
  f.read(reinterpret_cast<char*>(&magic), 8);
  f.read(reinterpret_cast<char*>(&n), 8);
  if (!f || magic != kTrieMagic) throw std::runtime_error("not a Full Block trie index: " + path);
  FullBlockTrie t;
  t.nodes_.resize(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    Node& node = t.nodes_[i];
    f.read(reinterpret_cast<char*>(&node.parent), 8);
    f.read(reinterpret_cast<char*>(&node.key), 8);
    f.read(reinterpret_cast<char*>(&node.record), 8);
    if (!f) throw std::runtime_error("truncated trie index: " + path);
    if (node.parent < -1 || node.parent >= static_cast<std::int64_t>(i))
      throw std::runtime_error("corrupt trie index (parent after child): " + path);
    if (!t.child_.emplace(std::make_pair(node.parent, node.key), static_cast<std::int64_t>(i)).second)
      throw std::runtime_error("corrupt trie index (duplicate edge): " + path);
  }
  return t;
}

void fill_full_block(const dp_kv_geom& g, std::uint64_t seed, std::int64_t page, void* dst) {
  const std::int64_t words = static_cast<std::int64_t>(g.n_layer) * g.block_tokens * g.bytes_per_token_layer / 8;
  auto* w = static_cast<std::uint64_t*>(dst);
  const std::uint64_t mix = seed * kSeedMul;
  for (std::int64_t i = 0; i < words; ++i)
    w[i] = splitmix64(((static_cast<std::uint64_t>(page) << 32) | static_cast<std::uint64_t>(i)) ^ mix);
}

FullBlockFile::FullBlockFile(const std::string& path, const dp_kv_geom& g, std::int64_t n_records,
                             bool create, bool direct)
    : path_(path), geom_(g), n_records_(n_records) {
  if (dp_geom_check(&g) != DP_OK) throw std::invalid_argument("FullBlockFile: bad geometry");
  if (n_records < 1) throw std::invalid_argument("FullBlockFile: n_records must be >= 1");
  record_bytes_ = static_cast<std::int64_t>(g.n_layer) * g.block_tokens * g.bytes_per_token_layer;
  stride_ = (record_bytes_ + kAlign - 1) / kAlign * kAlign;
  fd_ = ::open(path.c_str(), create ? (O_RDWR | O_CREAT | O_TRUNC) : O_RDWR, 0644);
  if (fd_ < 0 && !create) fd_ = ::open(path.c_str(), O_RDONLY);  // read-only tier: writes fail loudly
  if (fd_ < 0) io_error("cannot open", path);
  if (create) {
    if (::ftruncate(fd_, n_records_ * stride_) != 0) io_error("cannot size", path);
  } else {
    struct stat st {};
    if (::fstat(fd_, &st) != 0) io_error("cannot stat", path);
    if (st.st_size < n_records_ * stride_)
      throw std::runtime_error("Full Block file " + path + " holds fewer than " + std::to_string(n_records_) +
                               " records");
  }
  if (direct) fd_direct_ = ::open(path.c_str(), O_RDONLY | O_DIRECT);  // -1: buffered reads only
}

FullBlockFile::~FullBlockFile() {
  if (fd_direct_ >= 0) ::close(fd_direct_);
  if (fd_ >= 0) ::close(fd_);
}

void FullBlockFile::write(std::int64_t record, const void* src) {
  if (record < 0 || record >= n_records_) throw std::out_of_range("FullBlockFile::write: record out of range");
  const char* p = static_cast<const char*>(src);
  std::int64_t done = 0;
  while (done < record_bytes_) {
    const ssize_t n = ::pwrite(fd_, p + done, record_bytes_ - done, record * stride_ + done);
    if (n <= 0) io_error("short write to", path_);
    done += n;
  }
}

void FullBlockFile::write_bytes(std::int64_t record, std::int64_t offset, std::int64_t n, const void* src) {
  if (record < 0 || record >= n_records_ || offset < 0 || n < 0 || offset + n > record_bytes_)
    throw std::out_of_range("FullBlockFile::write_bytes: range out of the record");
  const char* p = static_cast<const char*>(src);
  std::int64_t done = 0;
  while (done < n) {
    const ssize_t k = ::pwrite(fd_, p + done, n - done, record * stride_ + offset + done);
    if (k <= 0) io_error("short write to", path_);
    done += k;
  }
}

void FullBlockFile::read(std::int64_t record, void* dst) const {
  if (record < 0 || record >= n_records_) throw std::out_of_range("FullBlockFile::read: record out of range");
  char* p = static_cast<char*>(dst);
  const bool aligned = (reinterpret_cast<std::uintptr_t>(dst) % kAlign) == 0 && record_bytes_ % kAlign == 0;
  const int fd = (fd_direct_ >= 0 && aligned) ? fd_direct_ : fd_;
  std::int64_t done = 0;
  while (done < record_bytes_) {
    const ssize_t n = ::pread(fd, p + done, record_bytes_ - done, record * stride_ + done);
    if (n <= 0) io_error("short read from", path_);
    done += n;
  }
}

void FullBlockFile::read_run(std::int64_t record, std::int64_t n, void* dst) const {
  if (n < 1) return;
  if (record < 0 || record + n > n_records_) throw std::out_of_range("FullBlockFile::read_run: records out of range");
  char* p = static_cast<char*>(dst);
  if (stride_ != record_bytes_) {
    for (std::int64_t i = 0; i < n; ++i) read(record + i, p + i * record_bytes_);
    return;
  }
  const bool aligned = (reinterpret_cast<std::uintptr_t>(dst) % kAlign) == 0;
  const int fd = (fd_direct_ >= 0 && aligned) ? fd_direct_ : fd_;
  const std::int64_t total = n * record_bytes_;
  std::int64_t done = 0;
  while (done < total) {
    const ssize_t got = ::pread(fd, p + done, total - done, record * stride_ + done);
    if (got <= 0) io_error("short read from", path_);
    done += got;
  }
}

void FullBlockFile::populate(std::uint64_t seed, int threads) {
  threads = std::max(1, threads);
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> err(threads);
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        std::vector<std::uint64_t> buf(static_cast<std::size_t>(record_bytes_ / 8));
        for (std::int64_t r = t; r < n_records_; r += threads) {
          fill_full_block(geom_, seed, r, buf.data());
          write(r, buf.data());
        }
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  if (::fsync(fd_) != 0) io_error("cannot fsync", path_);
}

}  // namespace dualpath
