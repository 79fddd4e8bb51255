// fmv_nccl_stub.cpp -- TEST TRANSPORT, not product code.
//
// A host-staged implementation of the NCCL API subset libfftmv_cuda uses
// (ncclGetUniqueId, ncclCommInitRank, ncclAllGather, ncclAllReduce,
// ncclBroadcast, ncclCommSplit, ncclCommDestroy, ncclCommAbort,
// ncclCommGetAsyncError, ncclGetErrorString). Loaded with
// FMV_NCCL_LIB=build/libfmv_nccl_stub.so it lets several processes share ONE
// GPU (real NCCL refuses two ranks on one device), so the library's
// partitioned entry points run at world size 2/4 on the one-GPU test pool.
//
// Ranks meet in a POSIX shared-memory segment named by the unique id. Every
// collective is synchronous: it waits for the caller's stream, stages the
// data through the segment (cudaMemcpy with UVA, or memcpy when no GPU is
// present so the CPU tests can drive it with host buffers), and returns. A
// rank that waits longer than FMV_STUB_TIMEOUT_S (default 60) seconds for its
// peers fails the collective with ncclRemoteError and records it as the
// communicator's asynchronous error, which exercises the library's error path.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

enum : int {
  kSuccess = 0,
  kUnhandledCuda = 1,
  kSystemError = 2,
  kInternalError = 3,
  kInvalidArgument = 4,
  kRemoteError = 6,
};
enum : int { kInt8 = 0, kUint8 = 1, kInt32 = 2, kUint32 = 3, kInt64 = 4, kUint64 = 5, kHalf = 6, kFloat = 7, kDouble = 8 };

constexpr int kMaxRanks = 64;
constexpr size_t kSlot = size_t(2) << 20;  // bytes staged per rank per round

struct Header {
  std::atomic<int> arrive;
  std::atomic<int> gen;
  long long meta[2 * kMaxRanks];  // ncclCommSplit (color, key) exchange
};

struct Comm {
  std::string name;
  int rank = 0, nranks = 1;
  int splits = 0;
  int async_err = 0;
  Header* hdr = nullptr;
  unsigned char* data = nullptr;
  size_t bytes = 0;
};

size_t seg_bytes(int nranks) { return (sizeof(Header) + 127) / 128 * 128 + (size_t)nranks * kSlot; }

bool have_cuda() {
  static const bool ok = [] {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
  }();
  return ok;
}

int copy(void* dst, const void* src, size_t n) {
  if (!n) return kSuccess;
  if (have_cuda()) return cudaMemcpy(dst, src, n, cudaMemcpyDefault) == cudaSuccess ? kSuccess : kUnhandledCuda;
  std::memcpy(dst, src, n);
  return kSuccess;
}

int stream_wait(cudaStream_t s) {
  if (!have_cuda()) return kSuccess;
  return cudaStreamSynchronize(s) == cudaSuccess ? kSuccess : kUnhandledCuda;
}

double timeout_s() {
  const char* v = getenv("FMV_STUB_TIMEOUT_S");
  return v && *v ? atof(v) : 60.0;
}

// Sense-reversing barrier over the segment.
int barrier(Comm* c) {
  if (c->nranks == 1) return kSuccess;
  Header* h = c->hdr;
  const int g = h->gen.load(std::memory_order_acquire);
  if (h->arrive.fetch_add(1, std::memory_order_acq_rel) + 1 == c->nranks) {
    h->arrive.store(0, std::memory_order_relaxed);
    h->gen.fetch_add(1, std::memory_order_acq_rel);
    return kSuccess;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const double lim = timeout_s();
  for (long it = 0; h->gen.load(std::memory_order_acquire) == g; ++it) {
    if (it < 1000) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(100));
    if ((it & 255) == 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > lim) {
      c->async_err = kRemoteError;
      return kRemoteError;
    }
  }
  return kSuccess;
}

size_t dsize(int dt) {
  switch (dt) {
    case kInt8: case kUint8: return 1;
    case kHalf: return 2;
    case kInt32: case kUint32: case kFloat: return 4;
    case kInt64: case kUint64: case kDouble: return 8;
    default: return 0;
  }
}

unsigned char* slot(Comm* c, int r) { return c->data + (size_t)r * kSlot; }

int open_comm(Comm* c, const std::string& name, int nranks, int rank) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return kInvalidArgument;
  c->name = name;
  c->rank = rank;
  c->nranks = nranks;
  c->bytes = seg_bytes(nranks);
  const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) return kSystemError;
  struct stat st{};
  if (fstat(fd, &st) != 0 || ((size_t)st.st_size < c->bytes && ftruncate(fd, (off_t)c->bytes) != 0)) {
    close(fd);
    return kSystemError;
  }
  void* p = mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return kSystemError;
  c->hdr = static_cast<Header*>(p);  // a fresh segment is zero-filled: barrier state 0
  c->data = static_cast<unsigned char*>(p) + (sizeof(Header) + 127) / 128 * 128;
  return barrier(c);  // everyone mapped
}

}  // namespace

extern "C" {

typedef struct {
  char internal[128];
} ncclUniqueId;

const char* ncclGetErrorString(int rc) {
  switch (rc) {
    case kSuccess: return "no error (stub)";
    case kUnhandledCuda: return "unhandled cuda error (stub)";
    case kSystemError: return "system error (stub: shared memory)";
    case kInvalidArgument: return "invalid argument (stub)";
    case kRemoteError: return "remote process exited or timed out (stub: FMV_STUB_TIMEOUT_S)";
    default: return "internal error (stub)";
  }
}

int ncclGetUniqueId(ncclUniqueId* id) {
  std::random_device rd;
  std::snprintf(id->internal, sizeof(id->internal), "/fmvstub-%d-%08x%08x", (int)getpid(), rd(), rd());
  return kSuccess;
}

int ncclCommInitRank(void** comm, int nranks, ncclUniqueId id, int rank) {
  auto* c = new Comm;
  const int rc = open_comm(c, std::string(id.internal, strnlen(id.internal, sizeof(id.internal))), nranks, rank);
  if (rc != kSuccess) {
    delete c;
    return rc;
  }
  *comm = c;
  return kSuccess;
}

int ncclCommGetAsyncError(void* comm, int* err) {
  *err = static_cast<Comm*>(comm)->async_err;
  return kSuccess;
}

int ncclCommDestroy(void* comm) {
  auto* c = static_cast<Comm*>(comm);
  if (!c) return kSuccess;
  if (c->hdr) munmap(c->hdr, c->bytes);
  shm_unlink(c->name.c_str());  // every rank has mapped it since init; ENOENT after the first is fine
  delete c;
  return kSuccess;
}

int ncclCommAbort(void* comm) { return ncclCommDestroy(comm); }

int ncclAllGather(const void* send, void* recv, size_t count, int dt, void* comm, cudaStream_t s) {
  auto* c = static_cast<Comm*>(comm);
  const size_t es = dsize(dt);
  if (!es) return kInvalidArgument;
  if (int rc = stream_wait(s)) return rc;
  const size_t total = count * es;
  for (size_t off = 0; off < total; off += kSlot) {
    const size_t n = std::min(kSlot, total - off);
    if (int rc = copy(slot(c, c->rank), static_cast<const unsigned char*>(send) + off, n)) return rc;
    if (int rc = barrier(c)) return rc;
    for (int r = 0; r < c->nranks; ++r)
      if (int rc = copy(static_cast<unsigned char*>(recv) + (size_t)r * total + off, slot(c, r), n)) return rc;
    if (int rc = barrier(c)) return rc;
  }
  return kSuccess;
}

int ncclBroadcast(const void* send, void* recv, size_t count, int dt, int root, void* comm, cudaStream_t s) {
  auto* c = static_cast<Comm*>(comm);
  const size_t es = dsize(dt);
  if (!es || root < 0 || root >= c->nranks) return kInvalidArgument;
  if (int rc = stream_wait(s)) return rc;
  const size_t total = count * es;
  for (size_t off = 0; off < total; off += kSlot) {
    const size_t n = std::min(kSlot, total - off);
    if (c->rank == root)
      if (int rc = copy(slot(c, 0), static_cast<const unsigned char*>(send) + off, n)) return rc;
    if (int rc = barrier(c)) return rc;
    if (int rc = copy(static_cast<unsigned char*>(recv) + off, slot(c, 0), n)) return rc;
    if (int rc = barrier(c)) return rc;
  }
  return kSuccess;
}

// Sum only (op 0), double or float, summed in rank order on every rank.
int ncclAllReduce(const void* send, void* recv, size_t count, int dt, int op, void* comm, cudaStream_t s) {
  auto* c = static_cast<Comm*>(comm);
  if (op != 0 || (dt != kDouble && dt != kFloat)) return kInvalidArgument;
  const size_t es = dsize(dt);
  if (int rc = stream_wait(s)) return rc;
  const size_t total = count * es;
  std::vector<unsigned char> acc, tmp;
  for (size_t off = 0; off < total; off += kSlot) {
    const size_t n = std::min(kSlot, total - off);
    if (int rc = copy(slot(c, c->rank), static_cast<const unsigned char*>(send) + off, n)) return rc;
    if (int rc = barrier(c)) return rc;
    acc.assign(slot(c, 0), slot(c, 0) + n);
    for (int r = 1; r < c->nranks; ++r) {
      const unsigned char* q = slot(c, r);
      if (dt == kDouble)
        for (size_t i = 0; i < n / 8; ++i) reinterpret_cast<double*>(acc.data())[i] += reinterpret_cast<const double*>(q)[i];
      else
        for (size_t i = 0; i < n / 4; ++i) reinterpret_cast<float*>(acc.data())[i] += reinterpret_cast<const float*>(q)[i];
    }
    if (int rc = barrier(c)) return rc;
    if (int rc = copy(static_cast<unsigned char*>(recv) + off, acc.data(), n)) return rc;
  }
  return kSuccess;
}

// color < 0 (NCCL_SPLIT_NOCOLOR): no new communicator.
int ncclCommSplit(void* comm, int color, int key, void** newcomm, void* /*config*/) {
  auto* c = static_cast<Comm*>(comm);
  const int split_no = c->splits++;
  c->hdr->meta[2 * c->rank] = color;
  c->hdr->meta[2 * c->rank + 1] = key;
  if (int rc = barrier(c)) return rc;
  std::vector<std::pair<long long, int>> members;  // (key, parent rank) of my color
  for (int r = 0; r < c->nranks; ++r)
    if (c->hdr->meta[2 * r] == color) members.push_back({c->hdr->meta[2 * r + 1], r});
  if (int rc = barrier(c)) return rc;  // meta may be reused by the next split
  if (color < 0) {
    *newcomm = nullptr;
    return kSuccess;
  }
  std::sort(members.begin(), members.end());
  int me = 0;
  for (size_t i = 0; i < members.size(); ++i)
    if (members[i].second == c->rank) me = (int)i;
  auto* n = new Comm;
  const std::string name = c->name + "-s" + std::to_string(split_no) + "c" + std::to_string(color);
  const int rc = open_comm(n, name, (int)members.size(), me);
  if (rc != kSuccess) {
    delete n;
    return rc;
  }
  *newcomm = n;
  return kSuccess;
}

}  // extern "C"
