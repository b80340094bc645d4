// f2: the reference's binary graph / feature / label files
// (graph.py:194-249) streamed straight into HBM.
//
// The reference loads a file into host numpy arrays (np.frombuffer + astype,
// graph.py:203-249), which at papers100M scale means ~36 GB of host copies
// before anything reaches a GPU.  Here the payload goes file -> pinned staging
// -> HBM in chunks: `threads` host threads pread chunk k+1 into one half of the
// staging buffer while the DMA engine copies chunk k from the other half, so
// the load runs at min(page-cache read, PCIe/C2C) bandwidth with no full host
// copy.  The on-disk integer types already match the device layout (u64
// indptr = int64, u32 indices = int32 once validated < n <= 2^31-1); labels
// are widened u32 -> int64 by a kernel; feature rows are copied contiguously
// and re-pitched to the padded device row by a kernel.  CsrGraph.validate / LabelVector checks
// run as device reductions into a flags word.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "common.cuh"
#include "salient_internal.h"

namespace sal {
namespace {

constexpr uint32_t kFormatVersion = 1;  // graph.py:17 FORMAT_VERSION

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// Read [off, off+len) of the file into dst with `threads` parallel preads.
int read_range(int fd, int64_t off, int64_t len, uint8_t* dst, int threads) {
  if (len <= 0) return SAL_OK;
  const int64_t min_part = 4 << 20;
  int t = threads < 1 ? 1 : threads;
  if ((int64_t)t * min_part > len) t = (int)((len + min_part - 1) / min_part);
  if (t < 1) t = 1;
  std::vector<int> rc(t, SAL_OK);
  auto work = [&](int i) {
    int64_t part = (len + t - 1) / t;
    part = (part + 4095) & ~int64_t(4095);
    int64_t a = (int64_t)i * part, b = a + part;
    if (b > len) b = len;
    while (a < b) {
      ssize_t r = pread(fd, dst + a, (size_t)(b - a), (off_t)(off + a));
      if (r < 0) {
        if (errno == EINTR) continue;
        rc[i] = SAL_EIO;
        return;
      }
      if (r == 0) {  // file shrank under us
        rc[i] = SAL_ETRUNC;
        return;
      }
      a += r;
    }
  };
  if (t == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    th.reserve(t);
    for (int i = 0; i < t; ++i) th.emplace_back(work, i);
    for (auto& x : th) x.join();
  }
  for (int r : rc)
    if (r != SAL_OK) return set_error(r, r == SAL_EIO ? "read failed: %s" : "file shrank while loading",
                                      strerror(errno));
  return SAL_OK;
}

// Double-buffered file -> pinned -> device pipeline over [off, off+len) in
// pieces of at most `piece` bytes (a multiple of the caller's unit); consume
// enqueues the device work for one piece on `st`.
int stream_range(int fd, int64_t off, int64_t len, int64_t piece, uint8_t* pinned, int64_t half,
                 int threads, cudaStream_t st,
                 const std::function<int(const uint8_t*, int64_t, int64_t)>& consume) {
  if (len <= 0) return SAL_OK;
  if (piece <= 0 || piece > half) return set_error(SAL_EINVAL, "staging buffer too small");
  cudaEvent_t ev[2];
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return set_error(SAL_ECUDA, "event create failed");
  bool used[2] = {false, false};
  int rc = SAL_OK;
  int k = 0;
  for (int64_t pos = 0; pos < len && rc == SAL_OK; pos += piece, ++k) {
    const int b = k & 1;
    const int64_t n = len - pos < piece ? len - pos : piece;
    if (used[b] && cudaEventSynchronize(ev[b]) != cudaSuccess) {
      rc = set_error(SAL_ECUDA, "copy failed: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    uint8_t* buf = pinned + b * half;
    rc = read_range(fd, off + pos, n, buf, threads);
    if (rc != SAL_OK) break;
    rc = consume(buf, pos, n);
    if (rc != SAL_OK) break;
    if (cudaEventRecord(ev[b], st) != cudaSuccess) rc = set_error(SAL_ECUDA, "event record failed");
    used[b] = true;
  }
  for (int b = 0; b < 2; ++b) {
    if (used[b]) cudaEventSynchronize(ev[b]);
    cudaEventDestroy(ev[b]);
  }
  return rc;
}

__global__ void widen_u32_kernel(const uint32_t* __restrict__ in, int64_t n,
                                 int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

__global__ void validate_csr_kernel(const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices, int64_t n, int64_t e,
                                    int32_t* __restrict__ flags) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0 && (indptr[0] != 0 || indptr[n] != e)) atomicOr(&flags[0], 1);
  bool dec = false, oob = false;
  for (int64_t i = tid; i < n; i += stride) dec |= indptr[i + 1] < indptr[i];
  for (int64_t i = tid; i < e; i += stride) {
    const int32_t v = indices[i];
    oob |= v < 0 || (int64_t)v >= n;
  }
  if (__any_sync(0xffffffffu, dec) && (threadIdx.x & 31) == 0) atomicOr(&flags[1], 1);
  if (__any_sync(0xffffffffu, oob) && (threadIdx.x & 31) == 0) atomicOr(&flags[2], 1);
}

__global__ void validate_labels_kernel(const int64_t* __restrict__ y, int64_t n, int64_t c,
                                       int32_t* __restrict__ flags) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= y[i] < 0 || y[i] >= c;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&flags[0], 1);
}

template <typename U>
__global__ void repitch_kernel(const U* __restrict__ in, int64_t rows, int64_t row_units,
                               U* __restrict__ out, int64_t pitch_units) {
  const int64_t total = rows * row_units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / row_units, c = i - r * row_units;
    out[r * pitch_units + c] = in[i];
  }
}

int grid_for(int64_t n);

int launch_repitch(const uint8_t* in, int64_t rows, int64_t row, uint8_t* out, int64_t pitch,
                   cudaStream_t st) {
  // widest unit dividing the row, the pitch and both base addresses
  int u = 16;
  while (u > 1 && (row % u || pitch % u || (uintptr_t)in % u || (uintptr_t)out % u)) u >>= 1;
  const int64_t units = rows * (row / u);
  const int g = grid_for(units);
  switch (u) {
    case 16: repitch_kernel<<<g, 256, 0, st>>>((const uint4*)in, rows, row / 16, (uint4*)out, pitch / 16); break;
    case 8: repitch_kernel<<<g, 256, 0, st>>>((const uint2*)in, rows, row / 8, (uint2*)out, pitch / 8); break;
    case 4: repitch_kernel<<<g, 256, 0, st>>>((const uint32_t*)in, rows, row / 4, (uint32_t*)out, pitch / 4); break;
    case 2: repitch_kernel<<<g, 256, 0, st>>>((const uint16_t*)in, rows, row / 2, (uint16_t*)out, pitch / 2); break;
    default: repitch_kernel<<<g, 256, 0, st>>>(in, rows, row, out, pitch); break;
  }
  return cudaGetLastError() == cudaSuccess ? SAL_OK : set_error(SAL_ECUDA, "repitch launch failed");
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

int open_checked(const char* path, const sal_file_header* h, Fd& f) {
  if (!path || !h) return set_error(SAL_EINVAL, "null path or header");
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return set_error(SAL_EIO, "%s: %s", path, strerror(errno));
  return SAL_OK;
}

}  // namespace
}  // namespace sal

extern "C" {

int sal_file_header_read(const char* path, int32_t kind, sal_file_header* out) {
  using sal::set_error;
  if (!path || !out) return set_error(SAL_EINVAL, "null argument");
  static const char* kMagic[4] = {nullptr, "MFGC", "FEAT", "LABL"};
  if (kind < SAL_FILE_CSR || kind > SAL_FILE_LABL) return set_error(SAL_EINVAL, "bad file kind %d", kind);
  memset(out, 0, sizeof(*out));
  out->kind = kind;
  sal::Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return set_error(SAL_EIO, "%s: %s", path, strerror(errno));
  struct stat sb;
  if (fstat(f.fd, &sb) != 0) return set_error(SAL_EIO, "%s: %s", path, strerror(errno));
  const int64_t size = (int64_t)sb.st_size;
  out->file_bytes = size;
  uint8_t hdr[24] = {0};
  const int64_t got = pread(f.fd, hdr, sizeof(hdr), 0);
  if (got < 0) return set_error(SAL_EIO, "%s: %s", path, strerror(errno));
  auto trunc = [&](const char* what) {
    return set_error(SAL_ETRUNC, "truncated file while reading %s", what);
  };
  // _check_header (graph.py:182-188): magic, then version
  if (got < 4) return trunc("magic");
  memcpy(out->magic, hdr, 4);
  if (memcmp(hdr, kMagic[kind], 4) != 0)
    return set_error(SAL_EBADMAGIC, "bad magic, expected %s", kMagic[kind]);
  if (got < 8) return trunc("version");
  uint32_t ver;
  memcpy(&ver, hdr + 4, 4);
  out->version = ver;
  if (ver != sal::kFormatVersion) return set_error(SAL_EVERSION, "unsupported version %u", ver);
  auto rd64 = [&](int o) { uint64_t v; memcpy(&v, hdr + o, 8); return v; };
  auto rd32 = [&](int o) { uint32_t v; memcpy(&v, hdr + o, 4); return v; };
  // payload extents; counts beyond any real file are reported as the
  // truncated field the reference's _read_exact would hit
  const uint64_t kHuge = 1ull << 60;
  if (kind == SAL_FILE_CSR) {  // load_csr (graph.py:202-214)
    if (got < 24) return trunc("counts");
    const uint64_t n = rd64(8), e = rd64(16);
    out->rows = (int64_t)n;
    out->cols = (int64_t)e;
    out->elem_bytes = 4;
    out->payload_offset = 24;
    if (n >= kHuge || (uint64_t)size < 24 + 8 * (n + 1)) return trunc("indptr");
    if (e >= kHuge || (uint64_t)size < 24 + 8 * (n + 1) + 4 * e) return trunc("indices");
  } else if (kind == SAL_FILE_FEAT) {  // load_features (graph.py:224-232)
    if (got < 24) return trunc("shape");
    const uint64_t rows = rd64(8);
    const uint32_t cols = rd32(16);
    const uint8_t code = hdr[20];
    out->rows = (int64_t)rows;
    out->cols = cols;
    out->dtype = code == SAL_F16 ? SAL_F16 : SAL_F32;  // any other code reads as f32
    out->elem_bytes = code == SAL_F16 ? 2 : 4;
    out->payload_offset = 24;
    if (rows >= kHuge || (uint64_t)size < 24 + rows * cols * (uint64_t)out->elem_bytes)
      return trunc("payload");
  } else {  // load_labels (graph.py:243-249)
    if (got < 20) return trunc("shape");
    const uint64_t rows = rd64(8);
    out->rows = (int64_t)rows;
    out->cols = rd32(16);
    out->elem_bytes = 4;
    out->payload_offset = 20;
    if (rows >= kHuge || (uint64_t)size < 20 + 4 * rows) return trunc("payload");
  }
  return SAL_OK;
}

int sal_load_csr(const char* path, const sal_file_header* h, int64_t* indptr_dev,
                 int32_t* indices_dev, void* pinned, int64_t pinned_bytes, int32_t threads,
                 void* stream) {
  using sal::set_error;
  sal::Fd f;
  int rc = sal::open_checked(path, h, f);
  if (rc) return rc;
  if (h->kind != SAL_FILE_CSR) return set_error(SAL_EINVAL, "header is not MFGC");
  if (h->rows >= (int64_t)INT32_MAX) return set_error(SAL_EINVAL, "device graphs hold < 2^31-1 nodes");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t half = (pinned_bytes / 2) & ~int64_t(4095);
  uint8_t* pin = (uint8_t*)pinned;
  const int64_t ip_bytes = 8 * (h->rows + 1), ix_bytes = 4 * h->cols;
  auto to = [&](uint8_t* dst) {
    return [=](const uint8_t* buf, int64_t pos, int64_t n) {
      return cudaMemcpyAsync(dst + pos, buf, n, cudaMemcpyHostToDevice, st) == cudaSuccess
                 ? SAL_OK
                 : set_error(SAL_ECUDA, "H2D copy failed");
    };
  };
  rc = sal::stream_range(f.fd, h->payload_offset, ip_bytes, half, pin, half, threads, st,
                         to((uint8_t*)indptr_dev));
  if (rc) return rc;
  return sal::stream_range(f.fd, h->payload_offset + ip_bytes, ix_bytes, half, pin, half, threads,
                           st, to((uint8_t*)indices_dev));
}

int sal_load_features(const char* path, const sal_file_header* h, void* out_dev,
                      int64_t out_stride_bytes, void* scratch_dev, void* pinned,
                      int64_t pinned_bytes, int32_t threads, void* stream) {
  using sal::set_error;
  sal::Fd f;
  int rc = sal::open_checked(path, h, f);
  if (rc) return rc;
  if (h->kind != SAL_FILE_FEAT) return set_error(SAL_EINVAL, "header is not FEAT");
  const int64_t row = h->cols * h->elem_bytes;
  if (out_stride_bytes < row) return set_error(SAL_EINVAL, "row pitch %lld < row bytes %lld",
                                               (long long)out_stride_bytes, (long long)row);
  if (row == 0 || h->rows == 0) return SAL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t half = (pinned_bytes / 2) & ~int64_t(4095);
  const int64_t piece = (half / row) * row;  // whole rows per chunk
  uint8_t* dst = (uint8_t*)out_dev;
  if (out_stride_bytes != row && !scratch_dev)
    return set_error(SAL_EINVAL, "padded row pitch needs a device scratch buffer");
  // a pitched H2D copy moves one small row per DMA descriptor (measured ~1.8 GB/s
  // for 200 B rows); instead each chunk lands contiguously in device scratch and
  // a kernel re-pitches it at HBM speed
  int launches = 0;
  int rc2 = sal::stream_range(
      f.fd, h->payload_offset, h->rows * row, piece, (uint8_t*)pinned, half, threads, st,
      [&](const uint8_t* buf, int64_t pos, int64_t n) {
        const int64_t r0 = pos / row, nr = n / row;
        if (out_stride_bytes == row)
          return cudaMemcpyAsync(dst + pos, buf, n, cudaMemcpyHostToDevice, st) == cudaSuccess
                     ? SAL_OK
                     : set_error(SAL_ECUDA, "H2D copy failed");
        if (cudaMemcpyAsync(scratch_dev, buf, n, cudaMemcpyHostToDevice, st) != cudaSuccess)
          return set_error(SAL_ECUDA, "H2D copy failed");
        ++launches;
        return sal::launch_repitch((const uint8_t*)scratch_dev, nr, row,
                                   dst + r0 * out_stride_bytes, out_stride_bytes, st);
      });
  sal::count_launch(launches);
  return rc2;
}

int sal_load_labels(const char* path, const sal_file_header* h, int64_t* out_dev,
                    void* scratch_dev, void* pinned, int64_t pinned_bytes, int32_t threads,
                    void* stream) {
  using sal::set_error;
  sal::Fd f;
  int rc = sal::open_checked(path, h, f);
  if (rc) return rc;
  if (h->kind != SAL_FILE_LABL) return set_error(SAL_EINVAL, "header is not LABL");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t half = (pinned_bytes / 2) & ~int64_t(4095);
  uint32_t* scratch = (uint32_t*)scratch_dev;
  int launches = 0;
  rc = sal::stream_range(
      f.fd, h->payload_offset, 4 * h->rows, half, (uint8_t*)pinned, half, threads, st,
      [&](const uint8_t* buf, int64_t pos, int64_t n) {
        if (cudaMemcpyAsync(scratch, buf, n, cudaMemcpyHostToDevice, st) != cudaSuccess)
          return set_error(SAL_ECUDA, "H2D copy failed");
        sal::widen_u32_kernel<<<sal::grid_for(n / 4), 256, 0, st>>>(scratch, n / 4,
                                                                    out_dev + pos / 4);
        ++launches;
        return cudaGetLastError() == cudaSuccess ? SAL_OK
                                                 : set_error(SAL_ECUDA, "widen launch failed");
      });
  sal::count_launch(launches);
  return rc;
}

int sal_validate_csr(const int64_t* indptr_dev, const int32_t* indices_dev, int64_t n, int64_t e,
                     int32_t* flags_dev, void* stream) {
  if (!indptr_dev || !flags_dev || n < 0 || e < 0)
    return sal::set_error(SAL_EINVAL, "validate_csr: invalid argument (!indptr_dev || !flags_dev || n < 0 || e < 0)");
  const int64_t m = n > e ? n : e;
  sal::validate_csr_kernel<<<sal::grid_for(m), 256, 0, (cudaStream_t)stream>>>(
      indptr_dev, indices_dev, n, e, flags_dev);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_validate_labels(const int64_t* y_dev, int64_t n, int64_t num_classes, int32_t* flags_dev,
                        void* stream) {
  if (!flags_dev || n < 0)
    return sal::set_error(SAL_EINVAL, "validate_labels: invalid argument (!flags_dev || n < 0)");
  if (n == 0) return SAL_OK;
  sal::validate_labels_kernel<<<sal::grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      y_dev, n, num_classes, flags_dev);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

}  // extern "C"
