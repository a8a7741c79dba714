// SSD tier I/O of the tier-move executor (include/kvt_b200.h):
// pinned host pieces <-> a file on local storage, O_DIRECT when the piece
// and its offset are 4 KiB aligned (the page cache would otherwise absorb
// the writes and the measured rate would be DRAM's), spread over worker
// threads that each take pieces from an atomic counter (the reference's
// work-queue pattern, proj/tools/kvtier_main.cpp:206-235). Host code only.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "kvt_b200.h"

namespace kvt {
int set_error(int code, const std::string& msg);
}

namespace {
constexpr int64_t kAlign = 4096;
constexpr int64_t kPiece = 64LL << 20;  // one pwrite / pread call moves at most this much

bool aligned(const void* p, int64_t n, int64_t off) {
  return (reinterpret_cast<uintptr_t>(p) % kAlign) == 0 && n % kAlign == 0 && off % kAlign == 0;
}

int run_io(int fd_direct, int fd_buffered, const kvt_file_io* ios, int64_t n, int32_t threads, bool write) {
  // split every request into <= kPiece chunks, hand them out from a counter
  struct Job {
    char* p;
    int64_t bytes, off;
  };
  std::vector<Job> jobs;
  for (int64_t i = 0; i < n; ++i) {
    if (ios[i].bytes < 0 || (ios[i].bytes > 0 && !ios[i].host) || ios[i].offset < 0)
      return kvt::set_error(KVT_EINVAL, "bad file io " + std::to_string(i));
    for (int64_t o = 0; o < ios[i].bytes; o += kPiece)
      jobs.push_back({static_cast<char*>(ios[i].host) + o, std::min(kPiece, ios[i].bytes - o), ios[i].offset + o});
  }
  std::atomic<size_t> next{0};
  std::atomic<int> err{0};
  auto worker = [&] {
    for (size_t j; (j = next.fetch_add(1)) < jobs.size() && !err.load();) {
      const Job& J = jobs[j];
      const int fd = (fd_direct >= 0 && aligned(J.p, J.bytes, J.off)) ? fd_direct : fd_buffered;
      int64_t done = 0;
      while (done < J.bytes) {
        const ssize_t r = write ? pwrite(fd, J.p + done, static_cast<size_t>(J.bytes - done), J.off + done)
                                : pread(fd, J.p + done, static_cast<size_t>(J.bytes - done), J.off + done);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) {
          err.store(r < 0 ? errno : EIO);
          return;
        }
        done += r;
      }
    }
  };
  const int nt = std::max(1, std::min<int>(threads, static_cast<int>(jobs.size())));
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  if (err.load()) return kvt::set_error(KVT_EINVAL, std::string(write ? "pwrite" : "pread") + ": " + std::strerror(err.load()));
  return KVT_OK;
}
}  // namespace

struct kvt_tier_file {
  int fd_direct = -1, fd_buffered = -1;
  bool direct = false;
};

extern "C" int kvt_tier_file_open(const char* path, int64_t bytes, kvt_tier_file** out) {
  if (!path || !out || bytes < 0) return kvt::set_error(KVT_EINVAL, "bad tier file request");
  auto* f = new kvt_tier_file();
  f->fd_buffered = ::open(path, O_RDWR | O_CREAT | O_TRUNC, 0600);
  if (f->fd_buffered < 0) {
    const std::string m = std::string("open ") + path + ": " + std::strerror(errno);
    delete f;
    return kvt::set_error(KVT_EINVAL, m);
  }
  if (bytes > 0 && posix_fallocate(f->fd_buffered, 0, bytes) != 0 && ftruncate(f->fd_buffered, bytes) != 0) {
    const std::string m = std::string("reserve ") + path + ": " + std::strerror(errno);
    ::close(f->fd_buffered);
    delete f;
    return kvt::set_error(KVT_EINVAL, m);
  }
  f->fd_direct = ::open(path, O_RDWR | O_DIRECT);  // some file systems (tmpfs, overlay) refuse O_DIRECT
  f->direct = f->fd_direct >= 0;
  *out = f;
  return KVT_OK;
}

extern "C" int kvt_tier_file_direct(const kvt_tier_file* f) { return f && f->direct ? 1 : 0; }

extern "C" int kvt_tier_file_close(kvt_tier_file* f) {
  if (!f) return KVT_OK;
  if (f->fd_direct >= 0) ::close(f->fd_direct);
  if (f->fd_buffered >= 0) ::close(f->fd_buffered);
  delete f;
  return KVT_OK;
}

extern "C" int kvt_tier_file_write(kvt_tier_file* f, const kvt_file_io* ios, int64_t n, int32_t threads) {
  if (!f || (n > 0 && !ios)) return kvt::set_error(KVT_EINVAL, "null argument");
  int rc = run_io(f->fd_direct, f->fd_buffered, ios, n, threads, true);
  if (rc == KVT_OK && fdatasync(f->fd_buffered) != 0)
    return kvt::set_error(KVT_EINVAL, std::string("fdatasync: ") + std::strerror(errno));
  return rc;
}

extern "C" int kvt_tier_file_read(kvt_tier_file* f, const kvt_file_io* ios, int64_t n, int32_t threads) {
  if (!f || (n > 0 && !ios)) return kvt::set_error(KVT_EINVAL, "null argument");
  return run_io(f->fd_direct, f->fd_buffered, ios, n, threads, false);
}
