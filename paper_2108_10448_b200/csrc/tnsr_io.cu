// tnsr_io.cu -- TNSR v1 tensor files streamed straight between disk and HBM
// (reference /root/reference/pkg/src/rtcur/tensorfile.py).
//
// Layout (little-endian): "TNSR" | u16 version (1) | u16 mode count n |
// n x u64 extents | prod(extents) IEEE-754 doubles, mode-1 fastest.
//
// The reference reads the whole payload with np.fromfile into host memory and
// writes it with a single-threaded tofile.  Here the payload moves in chunks
// through two pinned staging buffers: while chunk i is copied host->device
// (async on the caller's stream) chunk i+1 is read from the file by a few
// pread threads, so disk and PCIe overlap; a device kernel converts to fp32
// and/or extracts a mode-1 slab [lo, hi) on the fly (sharded loading).  The
// writer mirrors it (device fp32->fp64 + D2H of chunk i+1 while chunk i is
// pwritten).  Header validation reproduces the reference's checks and
// messages (byte offsets), so TensorFormatError texts match.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <thread>

namespace {

constexpr char kMagic[4] = {'T', 'N', 'S', 'R'};
constexpr int kVersion = 1;
constexpr i64 kChunk = (i64)64 << 20;   // bytes of fp64 payload per staging buffer
constexpr int kIoThreads = 4;

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// read exactly len bytes at off (false on short read / error)
bool pread_all(int fd, void* buf, size_t len, off_t off) {
  char* p = static_cast<char*>(buf);
  while (len > 0) {
    const ssize_t k = pread(fd, p, len, off);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      return false;
    }
    p += k;
    len -= (size_t)k;
    off += k;
  }
  return true;
}

bool pwrite_all(int fd, const void* buf, size_t len, off_t off) {
  const char* p = static_cast<const char*>(buf);
  while (len > 0) {
    const ssize_t k = pwrite(fd, p, len, off);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      return false;
    }
    p += k;
    len -= (size_t)k;
    off += k;
  }
  return true;
}

// split [off, off+len) over kIoThreads preads/pwrites
bool parallel_io(int fd, char* buf, size_t len, off_t off, bool write) {
  if (len < ((size_t)4 << 20)) return write ? pwrite_all(fd, buf, len, off) : pread_all(fd, buf, len, off);
  std::thread th[kIoThreads];
  bool ok[kIoThreads];
  const size_t part = (len / kIoThreads + 4095) & ~(size_t)4095;
  for (int t = 0; t < kIoThreads; ++t) {
    const size_t b = std::min(len, (size_t)t * part), e = std::min(len, (size_t)(t + 1) * part);
    ok[t] = true;
    if (e > b)
      th[t] = std::thread([&, t, b, e] {
        ok[t] = write ? pwrite_all(fd, buf + b, e - b, off + (off_t)b) : pread_all(fd, buf + b, e - b, off + (off_t)b);
      });
  }
  bool all = true;
  for (int t = 0; t < kIoThreads; ++t) {
    if (th[t].joinable()) th[t].join();
    all = all && ok[t];
  }
  return all;
}

std::string dims_str(const std::vector<unsigned long long>& d) {
  std::string s = "(";
  for (size_t i = 0; i < d.size(); ++i) {
    s += std::to_string(d[i]);
    if (d.size() == 1) s += ",";
    else if (i + 1 < d.size()) s += ", ";
  }
  return s + ")";
}

// exact decimal of 8 * prod(d) (Python int semantics, as the reference's
// "require {expected}" text): base-1e9 limbs, any number of u64 factors
std::string payload_bytes_str(const std::vector<unsigned long long>& d) {
  std::vector<unsigned long long> limbs{8};   // little-endian base 1e9
  const unsigned long long B = 1000000000ULL;
  for (unsigned long long f : d) {
    const unsigned long long parts[3] = {f % B, (f / B) % B, f / B / B};   // f = p0 + p1 B + p2 B^2
    std::vector<unsigned long long> acc(limbs.size() + 4, 0);
    for (int q = 0; q < 3; ++q) {
      unsigned __int128 carry = 0;
      size_t i = 0;
      for (; i < limbs.size(); ++i) {
        unsigned __int128 t = (unsigned __int128)limbs[i] * parts[q] + acc[i + q] + carry;
        acc[i + q] = (unsigned long long)(t % B);
        carry = t / B;
      }
      for (size_t k = i + q; carry; ++k) {
        unsigned __int128 t = acc[k] + carry;
        acc[k] = (unsigned long long)(t % B);
        carry = t / B;
      }
    }
    while (acc.size() > 1 && acc.back() == 0) acc.pop_back();
    limbs.swap(acc);
  }
  std::string out = std::to_string(limbs.back());
  for (size_t i = limbs.size() - 1; i-- > 0;) {
    std::string part = std::to_string(limbs[i]);
    out += std::string(9 - part.size(), '0') + part;
  }
  return out;
}

// tensorfile._parse_header (+ the payload-size check of read_tensor when check_payload)
int parse_header(const char* path, int* version, std::vector<i64>& dims, i64* payload_off, bool check_payload) {
  struct stat sb;
  if (stat(path, &sb) != 0) {
    if (errno == ENOENT) return fail(RT_ERR_NOTFOUND, std::string(path) + ": no such file");
    return fail(RT_ERR_IO, std::string(path) + ": " + strerror(errno));
  }
  const i64 size = (i64)sb.st_size;
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return fail(errno == ENOENT ? RT_ERR_NOTFOUND : RT_ERR_IO, std::string(path) + ": " + strerror(errno));
  const std::string P(path);
  if (size < 8)
    return fail(RT_ERR_FORMAT, P + ": file ends at byte " + std::to_string(size) + ", header needs at least 8 bytes");
  unsigned char h[8];
  if (!pread_all(f.fd, h, 8, 0)) return fail(RT_ERR_IO, P + ": read failed");
  if (memcmp(h, kMagic, 4) != 0) {
    std::string got = "b'";
    for (int i = 0; i < 4; ++i) {
      const unsigned char c = h[i];
      if (c == '\\' || c == '\'') { got += '\\'; got += (char)c; }
      else if (c >= 32 && c < 127) got += (char)c;
      else {
        char buf[8];
        snprintf(buf, sizeof(buf), "\\x%02x", c);
        got += buf;
      }
    }
    got += "'";
    return fail(RT_ERR_FORMAT, P + ": bad magic " + got + " at byte 0, expected b'TNSR'");
  }
  const int ver = h[4] | (h[5] << 8);
  const int n = h[6] | (h[7] << 8);
  if (ver != kVersion)
    return fail(RT_ERR_FORMAT, P + ": unsupported format version " + std::to_string(ver) + " at byte 4, expected " +
                                   std::to_string(kVersion));
  if (n < 1) return fail(RT_ERR_FORMAT, P + ": mode count 0 at byte 6");
  const i64 dims_end = 8 + 8 * (i64)n;
  if (size < dims_end)
    return fail(RT_ERR_FORMAT, P + ": file ends at byte " + std::to_string(size) + ", " + std::to_string(n) +
                                   " extents need bytes 8.." + std::to_string(dims_end - 1));
  std::vector<unsigned char> raw((size_t)8 * n);
  if (!pread_all(f.fd, raw.data(), raw.size(), 8)) return fail(RT_ERR_IO, P + ": read failed");
  std::vector<unsigned long long> ud(n, 0);
  for (int m = 0; m < n; ++m) {
    unsigned long long v = 0;
    for (int b = 7; b >= 0; --b) v = (v << 8) | raw[(size_t)8 * m + b];
    ud[m] = v;
    if (v == 0)
      return fail(RT_ERR_FORMAT, P + ": extent 0 for mode " + std::to_string(m + 1) + " at byte " +
                                     std::to_string(8 + 8 * m));
  }
  if (check_payload) {
    // 8 * prod(dims) == payload bytes, overflow-safe: test each factor against the
    // remaining headroom before multiplying (count <= 2^100, so count * d cannot wrap)
    const unsigned __int128 cap = (unsigned __int128)1 << 100;
    unsigned __int128 count = 1;
    bool big = false;
    for (int m = 0; m < n && !big; ++m) {
      if (count > cap / ud[m]) big = true;
      else count *= ud[m];
    }
    const i64 actual = size - dims_end;
    if (big || count * 8 != (unsigned __int128)actual)
      return fail(RT_ERR_FORMAT, P + ": payload at byte " + std::to_string(dims_end) + " holds " +
                                     std::to_string(actual) + " bytes, dims " + dims_str(ud) + " require " +
                                     payload_bytes_str(ud));
  }
  dims.assign(n, 0);
  for (int m = 0; m < n; ++m) {
    if (ud[m] >= (1ULL << 63))   // not representable as an int64 extent (the payload check rejects it first)
      return fail(RT_ERR_FORMAT, P + ": extent " + std::to_string(ud[m]) + " for mode " + std::to_string(m + 1) +
                                     " at byte " + std::to_string(8 + 8 * m) + " exceeds 2^63 - 1");
    dims[m] = (i64)ud[m];
  }
  *version = ver;
  *payload_off = dims_end;
  return RT_OK;
}

// staged fp64 payload elements [e0, e0 + cnt) -> X_slab (dtype), slab [lo, hi) of mode 1
template <typename T>
__global__ void k_tnsr_scatter(const double* __restrict__ src, i64 e0, i64 cnt, i64 d1, i64 lo, i64 hi,
                               T* __restrict__ dst) {
  const i64 w = hi - lo;
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < cnt; k += (i64)gridDim.x * blockDim.x) {
    const i64 e = e0 + k;
    const i64 R = e / d1, i1 = e - R * d1;
    if (i1 >= lo && i1 < hi) dst[(i1 - lo) + w * R] = (T)src[k];
  }
}

__global__ void k_f32_to_f64(const float* __restrict__ src, i64 cnt, double* __restrict__ dst) {
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < cnt; k += (i64)gridDim.x * blockDim.x)
    dst[k] = (double)src[k];
}

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  void* d = nullptr;   // device staging (conversion / slab)
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (p[i]) cudaFreeHost(p[i]);
    }
    if (d) cudaFree(d);
  }
};

}  // namespace

extern "C" int rtcur_tnsr_read_header(const char* path, int check_payload, int32_t* version, int32_t* n,
                                      int64_t* dims, int dims_cap, int64_t* payload_offset) {
  if (!path) return fail(RT_ERR_VALUE, "null path");
  int ver = 0;
  std::vector<i64> d;
  i64 off = 0;
  const int st = parse_header(path, &ver, d, &off, check_payload != 0);
  if (st) return st;
  if (version) *version = ver;
  if (n) *n = (int32_t)d.size();
  if (dims)
    for (int m = 0; m < (int)d.size() && m < dims_cap; ++m) dims[m] = d[m];
  if (payload_offset) *payload_offset = off;
  return RT_OK;
}

extern "C" int rtcur_tnsr_load(const char* path, int64_t slab_lo, int64_t slab_hi, int dtype, void* dst, void* stream) {
  if (!path || !dst) return fail(RT_ERR_VALUE, "null argument");
  int ver = 0;
  std::vector<i64> dims;
  i64 off = 0;
  int st = parse_header(path, &ver, dims, &off, true);
  if (st) return st;
  const i64 d1 = dims[0];
  i64 total = 1;
  for (i64 d : dims) total *= d;
  const i64 lo = slab_lo, hi = slab_hi < 0 ? d1 : slab_hi;
  if (lo < 0 || hi > d1 || lo >= hi) return fail(RT_ERR_VALUE, "slab outside mode 1");
  if (dtype != 0 && dtype != 1) return fail(RT_ERR_VALUE, "dtype must be f64 (0) or f32 (1)");
  const bool direct = dtype == 0 && lo == 0 && hi == d1;   // bytes land in place
  cudaStream_t s = (cudaStream_t)stream;
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return fail(RT_ERR_IO, std::string(path) + ": " + strerror(errno));
  Pinned pb;
  const i64 chunk_el = kChunk / 8;
  for (int i = 0; i < 2; ++i) {
    CK(cudaHostAlloc(&pb.p[i], (size_t)kChunk, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&pb.ev[i], cudaEventDisableTiming));
  }
  if (!direct) CK(cudaMalloc(&pb.d, (size_t)kChunk * 2));
  const i64 nchunks = (total + chunk_el - 1) / chunk_el;
  for (i64 c = 0; c < nchunks; ++c) {
    const int b = (int)(c & 1);
    const i64 e0 = c * chunk_el, cnt = std::min(chunk_el, total - e0);
    if (c >= 2) CK(cudaEventSynchronize(pb.ev[b]));   // buffer b's previous copy is done
    if (!parallel_io(f.fd, static_cast<char*>(pb.p[b]), (size_t)cnt * 8, (off_t)(off + e0 * 8), false))
      return fail(RT_ERR_IO, std::string(path) + ": payload read failed at byte " + std::to_string(off + e0 * 8));
    if (direct) {
      CK(cudaMemcpyAsync(static_cast<double*>(dst) + e0, pb.p[b], (size_t)cnt * 8, cudaMemcpyHostToDevice, s));
    } else {
      double* dstage = static_cast<double*>(pb.d) + (size_t)b * chunk_el;
      CK(cudaMemcpyAsync(dstage, pb.p[b], (size_t)cnt * 8, cudaMemcpyHostToDevice, s));
      const unsigned grid = (unsigned)std::min<i64>((cnt + 255) / 256, 148 * 16);
      if (dtype == 0) k_tnsr_scatter<double><<<grid, 256, 0, s>>>(dstage, e0, cnt, d1, lo, hi, (double*)dst);
      else k_tnsr_scatter<float><<<grid, 256, 0, s>>>(dstage, e0, cnt, d1, lo, hi, (float*)dst);
      LAUNCH_CHECK();
    }
    CK(cudaEventRecord(pb.ev[b], s));
  }
  CK(cudaStreamSynchronize(s));
  return RT_OK;
}

extern "C" int rtcur_tnsr_store(const char* path, int n, const int64_t* dims, int dtype, const void* src, void* stream) {
  if (!path || !dims || !src || n < 1 || n > 65535) return fail(RT_ERR_VALUE, "bad arguments");
  if (dtype != 0 && dtype != 1) return fail(RT_ERR_VALUE, "dtype must be f64 (0) or f32 (1)");
  i64 total = 1;
  for (int m = 0; m < n; ++m) {
    if (dims[m] < 1) return fail(RT_ERR_VALUE, "extents must be positive");
    total *= dims[m];
  }
  cudaStream_t s = (cudaStream_t)stream;
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (f.fd < 0) return fail(RT_ERR_IO, std::string(path) + ": " + strerror(errno));
  std::vector<unsigned char> head((size_t)8 + 8 * n);
  memcpy(head.data(), kMagic, 4);
  head[4] = (unsigned char)(kVersion & 0xff);
  head[5] = (unsigned char)(kVersion >> 8);
  head[6] = (unsigned char)(n & 0xff);
  head[7] = (unsigned char)(n >> 8);
  for (int m = 0; m < n; ++m)
    for (int b = 0; b < 8; ++b) head[(size_t)8 + 8 * m + b] = (unsigned char)(((unsigned long long)dims[m] >> (8 * b)) & 0xff);
  if (!pwrite_all(f.fd, head.data(), head.size(), 0)) return fail(RT_ERR_IO, std::string(path) + ": header write failed");
  const i64 off = (i64)head.size();
  Pinned pb;
  const i64 chunk_el = kChunk / 8;
  for (int i = 0; i < 2; ++i) {
    CK(cudaHostAlloc(&pb.p[i], (size_t)kChunk, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&pb.ev[i], cudaEventDisableTiming));
  }
  if (dtype == 1) CK(cudaMalloc(&pb.d, (size_t)kChunk * 2));
  const i64 nchunks = (total + chunk_el - 1) / chunk_el;
  auto issue = [&](i64 c) -> int {
    const int b = (int)(c & 1);
    const i64 e0 = c * chunk_el, cnt = std::min(chunk_el, total - e0);
    const void* from = static_cast<const double*>(src) + e0;
    if (dtype == 1) {
      double* dstage = static_cast<double*>(pb.d) + (size_t)b * chunk_el;
      const unsigned grid = (unsigned)std::min<i64>((cnt + 255) / 256, 148 * 16);
      k_f32_to_f64<<<grid, 256, 0, s>>>(static_cast<const float*>(src) + e0, cnt, dstage);
      LAUNCH_CHECK();
      from = dstage;
    }
    CK(cudaMemcpyAsync(pb.p[b], from, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(pb.ev[b], s));
    return RT_OK;
  };
  if (nchunks > 0) {
    const int ist = issue(0);
    if (ist) return ist;
  }
  for (i64 c = 0; c < nchunks; ++c) {
    const int b = (int)(c & 1);
    const i64 e0 = c * chunk_el, cnt = std::min(chunk_el, total - e0);
    CK(cudaEventSynchronize(pb.ev[b]));
    if (c + 1 < nchunks) {   // the next chunk's D2H overlaps this chunk's write
      const int ist = issue(c + 1);
      if (ist) return ist;
    }
    if (!parallel_io(f.fd, static_cast<char*>(pb.p[b]), (size_t)cnt * 8, (off_t)(off + e0 * 8), true))
      return fail(RT_ERR_IO, std::string(path) + ": payload write failed at byte " + std::to_string(off + e0 * 8));
  }
  return RT_OK;
}
