// ssf_io.cpp — SSF1 trace files in, SMB1 pick files out.
//
// The reference reads a whole SSF1 file into a Dataset of per-trace vectors
// (io.hpp:124-166) and writes SMB1 picks from SemblanceMatrix results
// (io.hpp:170-194).  Here the formats are re-implemented for the GPU path:
//
//  * velan_ssf1_open indexes the file (one pass over the gather headers,
//    seeking over the samples) with read_dataset's validation and messages;
//  * velan_ssf1_read fills a block of gathers straight into the flattened
//    [G][fold][ns] layout of velan_gpu_dataset (pinned host memory when the
//    caller allocated it so), one pread per trace run, several threads;
//  * velan_ssf1_write / velan_smb1_write produce files byte-identical to
//    write_dataset (io.hpp:95-122) and write_picks (io.hpp:170-194);
//  * velan_smb1_begin / _append / _end stream SMB1 records block by block
//    (results never need to exist for the whole line at once).
//
// Little-endian hosts only (the formats are little-endian, io.hpp:20-22;
// x86-64 and aarch64 GPU hosts are).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/velan_gpu.h"

namespace velan_gpu {
void set_last_error(const std::string& msg);  // velan_gpu.cu
}

namespace {

struct IoError : std::runtime_error {
  int code;
  IoError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// velan::format_error (error.hpp) carries the byte offset in its message
std::string at_offset(const std::string& what, uint64_t off) {
  return what + " at byte " + std::to_string(off);
}

class File {
 public:
  File(const char* path, int flags, const char* what) : path_(path ? path : "") {
    fd_ = ::open(path_.c_str(), flags | O_CLOEXEC, 0644);
    if (fd_ < 0)
      throw IoError(VELAN_GPU_ERUNTIME, std::string(what) + path_ + ": " + std::strerror(errno));
  }
  ~File() {
    if (fd_ >= 0) ::close(fd_);
  }
  File(const File&) = delete;
  File& operator=(const File&) = delete;
  int fd() const { return fd_; }
  uint64_t size() const {
    struct stat st;
    if (::fstat(fd_, &st) != 0) throw IoError(VELAN_GPU_ERUNTIME, "fstat failed: " + path_);
    return static_cast<uint64_t>(st.st_size);
  }
  void pread_all(void* dst, uint64_t n, uint64_t off) const {
    char* p = static_cast<char*>(dst);
    while (n > 0) {
      const ssize_t r = ::pread(fd_, p, n, static_cast<off_t>(off));
      if (r < 0) {
        if (errno == EINTR) continue;
        throw IoError(VELAN_GPU_ERUNTIME, "read failed: " + path_ + ": " + std::strerror(errno));
      }
      if (r == 0) throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file", off));
      p += r;
      n -= static_cast<uint64_t>(r);
      off += static_cast<uint64_t>(r);
    }
  }
  void write_all(const void* src, uint64_t n) {
    const char* p = static_cast<const char*>(src);
    while (n > 0) {
      const ssize_t r = ::write(fd_, p, n);
      if (r < 0) {
        if (errno == EINTR) continue;
        throw IoError(VELAN_GPU_ERUNTIME, "write failed: " + path_ + ": " + std::strerror(errno));
      }
      p += r;
      n -= static_cast<uint64_t>(r);
    }
  }

 private:
  std::string path_;
  int fd_ = -1;
};

// Little-endian byte buffer with the reference writer's field order.
struct Bytes {
  std::vector<char> b;
  void u32(uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(static_cast<char>(v >> (8 * i)));
  }
  void f32(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    u32(u);
  }
  void raw(const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    b.insert(b.end(), c, c + n);
  }
  void f32s(const float* p, size_t n) { raw(p, 4 * n); }  // little-endian host
};

uint32_t le32(const unsigned char* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
         (static_cast<uint32_t>(p[2]) << 16) | (static_cast<uint32_t>(p[3]) << 24);
}

}  // namespace

struct velan_ssf1 {
  File file;
  velan_ssf1_info info{};
  std::vector<uint32_t> cdp_id, ntraces, ns, dt_us;
  std::vector<uint64_t> offset;  // byte offset of each gather's first trace
  uint64_t meta_off = 0;
  explicit velan_ssf1(const char* path) : file(path, O_RDONLY, "cannot open for reading: ") {}
};

namespace {

// read_dataset (io.hpp:124-166): magic, version, ncdps, fold; per gather the
// four header words, trace count <= fold, dt != 0; optional metadata tail;
// no trailing bytes.  The samples are skipped, not read.
void index_file(velan_ssf1& f) {
  const uint64_t size = f.file.size();
  unsigned char h[16];
  if (size < 4) throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file reading magic", 0));
  f.file.pread_all(h, 4, 0);
  if (std::memcmp(h, "SSF1", 4) != 0)
    throw IoError(VELAN_GPU_ECONFIG, at_offset("bad magic, expected SSF1", 0));
  if (size < 16) throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file reading header", 4));
  f.file.pread_all(h, 12, 4);
  const uint32_t version = le32(h);
  if (version != 1)
    throw IoError(VELAN_GPU_ECONFIG, at_offset("unsupported version " + std::to_string(version), 4));
  const uint32_t ncdps = le32(h + 4);
  const uint32_t fold = le32(h + 8);
  uint64_t off = 16;
  f.cdp_id.resize(ncdps);
  f.ntraces.resize(ncdps);
  f.ns.resize(ncdps);
  f.dt_us.resize(ncdps);
  f.offset.resize(ncdps);
  bool uniform = true;
  for (uint32_t g = 0; g < ncdps; ++g) {
    if (size - off < 16)
      throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file reading gather header", off));
    f.file.pread_all(h, 16, off);
    f.cdp_id[g] = le32(h);
    f.ntraces[g] = le32(h + 4);
    f.ns[g] = le32(h + 8);
    f.dt_us[g] = le32(h + 12);
    if (f.ntraces[g] > fold)
      throw IoError(VELAN_GPU_ECONFIG,
                    at_offset("gather " + std::to_string(f.cdp_id[g]) +
                                  " has more traces than fold",
                              off + 4));
    if (f.dt_us[g] == 0)
      throw IoError(VELAN_GPU_ECONFIG,
                    at_offset("gather " + std::to_string(f.cdp_id[g]) + " has dt 0", off + 12));
    off += 16;
    f.offset[g] = off;
    const uint64_t bytes = static_cast<uint64_t>(f.ntraces[g]) * (16 + 4ull * f.ns[g]);
    if (size - off < bytes)
      throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file reading traces", off));
    off += bytes;
    if (g > 0 && (f.ns[g] != f.ns[0] || f.dt_us[g] != f.dt_us[0])) uniform = false;
  }
  uint64_t meta = 0;
  if (size > off) {
    if (size - off < 4)
      throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file reading metadata length", off));
    f.file.pread_all(h, 4, off);
    meta = le32(h);
    off += 4;
    if (size - off < meta)
      throw IoError(VELAN_GPU_ECONFIG, at_offset("truncated file reading metadata", off));
    f.meta_off = off;
    off += meta;
    if (off != size) throw IoError(VELAN_GPU_ECONFIG, at_offset("trailing bytes after metadata", off));
  }
  f.info.n_gathers = ncdps;
  f.info.fold = fold;
  f.info.ns = ncdps ? f.ns[0] : 0;
  f.info.dt_us = ncdps ? f.dt_us[0] : 0;
  f.info.uniform = uniform ? 1 : 0;
  f.info.metadata_bytes = meta;
  f.info.file_bytes = size;
}

int fail(const IoError& e) {
  velan_gpu::set_last_error(e.what());
  return e.code;
}

}  // namespace

struct velan_smb1_writer {
  File file;
  uint32_t declared = 0, written = 0;
  int32_t ns = 0, nc = 0, with_matrix = 0;
  explicit velan_smb1_writer(const char* path)
      : file(path, O_WRONLY | O_CREAT | O_TRUNC, "cannot open for writing: ") {}
};

#define IO_BEGIN try {
#define IO_END                                        \
  }                                                   \
  catch (const IoError& e) {                          \
    return fail(e);                                   \
  }                                                   \
  catch (const std::exception& e) {                   \
    velan_gpu::set_last_error(e.what());              \
    return VELAN_GPU_ERUNTIME;                        \
  }

extern "C" {

int velan_ssf1_open(const char* path, velan_ssf1** out, velan_ssf1_info* info) {
  IO_BEGIN
  if (!path || !out) throw IoError(VELAN_GPU_EPARAM, "null path or handle");
  *out = nullptr;
  auto* f = new velan_ssf1(path);
  try {
    index_file(*f);
  } catch (...) {
    delete f;
    throw;
  }
  if (info) *info = f->info;
  *out = f;
  return VELAN_GPU_OK;
  IO_END
}

void velan_ssf1_close(velan_ssf1* f) { delete f; }

int velan_ssf1_gathers(const velan_ssf1* f, uint32_t* cdp_id, int32_t* ntraces,
                       uint32_t* ns, uint32_t* dt_us) {
  IO_BEGIN
  if (!f) throw IoError(VELAN_GPU_EPARAM, "null handle");
  const size_t G = f->cdp_id.size();
  for (size_t g = 0; g < G; ++g) {
    if (cdp_id) cdp_id[g] = f->cdp_id[g];
    if (ntraces) ntraces[g] = static_cast<int32_t>(f->ntraces[g]);
    if (ns) ns[g] = f->ns[g];
    if (dt_us) dt_us[g] = f->dt_us[g];
  }
  return VELAN_GPU_OK;
  IO_END
}

int velan_ssf1_metadata(const velan_ssf1* f, char* buf, uint64_t cap) {
  IO_BEGIN
  if (!f) throw IoError(VELAN_GPU_EPARAM, "null handle");
  if (f->info.metadata_bytes > cap) throw IoError(VELAN_GPU_EPARAM, "metadata buffer too small");
  if (f->info.metadata_bytes) f->file.pread_all(buf, f->info.metadata_bytes, f->meta_off);
  return VELAN_GPU_OK;
  IO_END
}

}  // extern "C"

namespace {

// Gathers list[i] (or first + i when list is null), i < count, into the
// flattened layout: one pread of each gather's whole trace run.
void read_gathers(const velan_ssf1* f, const int32_t* list, int32_t first, int32_t count,
                  int32_t max_traces, float* samples, float* coords, int32_t n_threads) {
  if (!f->info.uniform)
    throw IoError(VELAN_GPU_ECONFIG,
                  "gathers differ in ns or dt_us: the flattened layout needs one ns");
  if (max_traces < static_cast<int32_t>(f->info.fold))
    throw IoError(VELAN_GPU_EPARAM, "max_traces smaller than the file's fold");
  const int ns = static_cast<int>(f->info.ns);
  const size_t stride = static_cast<size_t>(max_traces);
  // one pread of a gather's whole trace run into a scratch record buffer,
  // then split into coords and samples (records are 16 + 4 ns bytes)
  const int T = std::max(1, std::min<int>(n_threads > 0 ? n_threads
                                                        : static_cast<int>(std::thread::hardware_concurrency()),
                                          std::max(count, 1)));
  std::atomic<int> next{0};
  std::atomic<bool> failed{false};
  std::string err;
  int err_code = VELAN_GPU_OK;
  std::atomic_flag err_lock = ATOMIC_FLAG_INIT;
  auto work = [&]() {
    std::vector<unsigned char> rec;
    for (int i = next++; i < count && !failed; i = next++) {
      const int g = list ? list[i] : first + i;
      const uint32_t M = f->ntraces[g];
      const size_t rb = 16 + 4ull * ns;
      rec.resize(rb * M);
      try {
        if (M) f->file.pread_all(rec.data(), rb * M, f->offset[g]);
      } catch (const IoError& e) {
        while (err_lock.test_and_set()) {
        }
        if (!failed) {
          err = e.what();
          err_code = e.code;
          failed = true;
        }
        err_lock.clear();
        return;
      }
      float* sg = samples + static_cast<size_t>(i) * stride * ns;
      float* cg = coords + static_cast<size_t>(i) * stride * 4;
      for (uint32_t m = 0; m < M; ++m) {
        const unsigned char* r = rec.data() + rb * m;
        std::memcpy(cg + 4 * m, r, 16);
        std::memcpy(sg + static_cast<size_t>(m) * ns, r + 16, 4ull * ns);
      }
      // traces beyond the gather's count: zero (the layout's padding)
      std::memset(cg + 4 * M, 0, 16 * (stride - M));
      std::memset(sg + static_cast<size_t>(M) * ns, 0, 4ull * ns * (stride - M));
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  if (failed) throw IoError(err_code, err);
}

}  // namespace

extern "C" {

int velan_ssf1_read(const velan_ssf1* f, int32_t first, int32_t count, int32_t max_traces,
                    float* samples, float* coords, int32_t n_threads) {
  IO_BEGIN
  if (!f || !samples || !coords) throw IoError(VELAN_GPU_EPARAM, "null handle or buffer");
  if (first < 0 || count < 0 || static_cast<uint64_t>(first) + count > f->cdp_id.size())
    throw IoError(VELAN_GPU_EPARAM, "gather range outside the file");
  read_gathers(f, nullptr, first, count, max_traces, samples, coords, n_threads);
  return VELAN_GPU_OK;
  IO_END
}

int velan_ssf1_read_list(const velan_ssf1* f, const int32_t* gathers, int32_t count,
                         int32_t max_traces, float* samples, float* coords,
                         int32_t n_threads) {
  IO_BEGIN
  if (!f || !samples || !coords || (count > 0 && !gathers))
    throw IoError(VELAN_GPU_EPARAM, "null handle or buffer");
  if (count < 0) throw IoError(VELAN_GPU_EPARAM, "count < 0");
  for (int32_t i = 0; i < count; ++i)
    if (gathers[i] < 0 || static_cast<uint64_t>(gathers[i]) >= f->cdp_id.size())
      throw IoError(VELAN_GPU_EPARAM, "gather index outside the file");
  read_gathers(f, gathers, 0, count, max_traces, samples, coords, n_threads);
  return VELAN_GPU_OK;
  IO_END
}

int velan_ssf1_midpoints(const velan_ssf1* f, float* mx, float* my) {
  IO_BEGIN
  if (!f || !mx || !my) throw IoError(VELAN_GPU_EPARAM, "null handle or buffer");
  const size_t G = f->cdp_id.size();
  unsigned char h[16];
  for (size_t g = 0; g < G; ++g) {
    // midpoint_of (types.hpp:57-62): the first trace's source and receiver
    if (f->ntraces[g] == 0)
      throw IoError(VELAN_GPU_EPARAM, "midpoint_of: gather " + std::to_string(f->cdp_id[g]) +
                                          " has no traces");
    f->file.pread_all(h, 16, f->offset[g]);
    float c[4];
    std::memcpy(c, h, 16);  // little-endian host
    mx[g] = (c[0] + c[2]) * 0.5f;
    my[g] = (c[1] + c[3]) * 0.5f;
  }
  return VELAN_GPU_OK;
  IO_END
}

int velan_ssf1_write(const char* path, const velan_gpu_dataset* ds, const char* metadata,
                     uint64_t metadata_bytes) {
  IO_BEGIN
  if (!path || !ds) throw IoError(VELAN_GPU_EPARAM, "null path or dataset");
  if (ds->samples_mem != VELAN_MEM_HOST)
    throw IoError(VELAN_GPU_EPARAM, "velan_ssf1_write: samples must be host memory");
  File out(path, O_WRONLY | O_CREAT | O_TRUNC, "cannot open for writing: ");
  Bytes b;
  b.raw("SSF1", 4);
  b.u32(1);
  b.u32(static_cast<uint32_t>(ds->n_gathers));
  b.u32(static_cast<uint32_t>(ds->max_traces));
  out.write_all(b.b.data(), b.b.size());
  const size_t ns = static_cast<size_t>(ds->ns);
  for (int g = 0; g < ds->n_gathers; ++g) {
    // write_dataset's check (io.hpp:101-104)
    if (ds->ntraces[g] > ds->max_traces || ds->ntraces[g] < 0)
      throw IoError(VELAN_GPU_EPARAM,
                    "write_dataset: gather " + std::to_string(ds->cdp_id[g]) + " exceeds fold");
    b.b.clear();
    b.u32(ds->cdp_id[g]);
    b.u32(static_cast<uint32_t>(ds->ntraces[g]));
    b.u32(static_cast<uint32_t>(ds->ns));
    b.u32(ds->dt_us);
    for (int m = 0; m < ds->ntraces[g]; ++m) {
      const size_t t = static_cast<size_t>(g) * ds->max_traces + m;
      b.f32s(ds->coords + 4 * t, 4);
      b.f32s(ds->samples + t * ns, ns);
    }
    out.write_all(b.b.data(), b.b.size());
  }
  if (metadata_bytes > 0) {
    b.b.clear();
    b.u32(static_cast<uint32_t>(metadata_bytes));
    b.raw(metadata, metadata_bytes);
    out.write_all(b.b.data(), b.b.size());
  }
  return VELAN_GPU_OK;
  IO_END
}

int velan_smb1_begin(const char* path, uint32_t n_cdps, int32_t ns, int32_t nc,
                     int32_t with_matrix, velan_smb1_writer** out) {
  IO_BEGIN
  if (!path || !out) throw IoError(VELAN_GPU_EPARAM, "null path or handle");
  if (ns < 0 || nc < 0) throw IoError(VELAN_GPU_EPARAM, "negative ns or nc");
  auto* w = new velan_smb1_writer(path);
  w->declared = n_cdps;
  w->ns = ns;
  w->nc = nc;
  w->with_matrix = with_matrix ? 1 : 0;
  Bytes b;
  b.raw("SMB1", 4);
  b.u32(1);
  b.u32(n_cdps);
  b.u32(with_matrix ? 1u : 0u);
  try {
    w->file.write_all(b.b.data(), b.b.size());
  } catch (...) {
    delete w;
    throw;
  }
  *out = w;
  return VELAN_GPU_OK;
  IO_END
}

int velan_smb1_append(velan_smb1_writer* w, int32_t n, const uint32_t* cdp_id,
                      const float* pick_velocity, const float* pick_semblance,
                      const float* matrix) {
  IO_BEGIN
  if (!w || (n > 0 && (!cdp_id || !pick_velocity || !pick_semblance)))
    throw IoError(VELAN_GPU_EPARAM, "null writer or pick arrays");
  if (w->with_matrix && n > 0 && !matrix)
    throw IoError(VELAN_GPU_EPARAM, "matrix flagged but not given");
  if (static_cast<uint64_t>(w->written) + n > w->declared)
    throw IoError(VELAN_GPU_EPARAM, "more records than declared");
  const size_t ns = static_cast<size_t>(w->ns), nc = static_cast<size_t>(w->nc);
  Bytes b;
  for (int r = 0; r < n; ++r) {
    b.b.clear();
    b.u32(cdp_id[r]);
    b.u32(static_cast<uint32_t>(w->ns));
    b.u32(static_cast<uint32_t>(w->nc));
    for (size_t k = 0; k < ns; ++k) {  // ns x (velocity, semblance)
      b.f32(pick_velocity[r * ns + k]);
      b.f32(pick_semblance[r * ns + k]);
    }
    w->file.write_all(b.b.data(), b.b.size());
    if (w->with_matrix) w->file.write_all(matrix + r * ns * nc, 4 * ns * nc);
  }
  w->written += static_cast<uint32_t>(n);
  return VELAN_GPU_OK;
  IO_END
}

int velan_smb1_end(velan_smb1_writer* w) {
  if (!w) return VELAN_GPU_EPARAM;
  const bool complete = w->written == w->declared;
  delete w;
  if (!complete) {
    velan_gpu::set_last_error("SMB1 writer closed before all declared records were written");
    return VELAN_GPU_EPARAM;
  }
  return VELAN_GPU_OK;
}

}  // extern "C"
