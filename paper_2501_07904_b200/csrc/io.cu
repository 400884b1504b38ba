// Files straight to and from the device (SURVEY.md 8(f) "I/O straight to device"): the
// reference's binary containers (include/ttutv/io.hpp:10-19, src/io.cpp:139-211),
//   TTUTVTEN: magic | u32 version=1 | u32 order | u64 dims[order] | f64 payload
//   TTUTVCOR: magic | u32 version=1 | u32 order | u64 ranks[order+1] | u64 dims[order]
//             | core payloads back to back,
// all little-endian. The reference slurps the whole file into a host string and copies
// it into a std::vector; here the payload streams through two pinned buffers, the file
// read of one chunk overlapping the H2D copy of the previous one, so an 8.6 GB tensor
// (config 5) never has a host copy. Header checks, messages and byte offsets are the
// reference's (src/io.cpp:35-137), so the C++ layer can rethrow ParseError(msg, offset).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <sys/stat.h>

#include "io.hpp"

namespace ttg {
namespace {

thread_local int64_t t_parse_offset = 0;

[[noreturn]] void parse_error(const std::string& msg, int64_t offset) {
    t_parse_offset = offset;
    fail(3, msg);
}

constexpr char kTensorMagic[9] = "TTUTVTEN";
constexpr char kTrainMagic[9] = "TTUTVCOR";
constexpr uint32_t kFileVersion = 1;
constexpr size_t kChunk = size_t(64) << 20;  // pinned staging buffer (bytes)

bool little_endian() {
    const uint16_t one = 1;
    unsigned char b = 0;
    std::memcpy(&b, &one, 1);
    return b == 1;
}

struct File {
    std::FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// The header bytes (at most 16 + 8 * 255), read with the reference's bounds checks.
class HeaderReader {
public:
    HeaderReader(std::vector<unsigned char> bytes, int64_t file_size, std::string path)
        : b_(std::move(bytes)), size_(file_size), path_(std::move(path)) {}
    int64_t offset() const { return pos_; }
    int64_t remaining() const { return size_ - pos_; }
    void expect_magic(const char* magic) {
        if (size_ < 8 || (int64_t)b_.size() < 8 || std::memcmp(b_.data(), magic, 8) != 0)
            parse_error(path_ + ": bad magic, not a recognized container", 0);
        pos_ += 8;
    }
    uint32_t u32(const char* what) {
        require(4, what);
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= (uint32_t)b_[(size_t)pos_ + i] << (8 * i);
        pos_ += 4;
        return v;
    }
    uint64_t u64(const char* what) {
        require(8, what);
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= (uint64_t)b_[(size_t)pos_ + i] << (8 * i);
        pos_ += 8;
        return v;
    }

private:
    void require(int64_t n, const char* what) {
        if (remaining() < n || pos_ + n > (int64_t)b_.size())
            parse_error(path_ + ": truncated header while reading " + what, pos_);
    }
    std::vector<unsigned char> b_;
    int64_t size_;
    std::string path_;
    int64_t pos_ = 0;
};

HeaderReader open_header(const std::string& path, File& file) {
    file.f = std::fopen(path.c_str(), "rb");
    if (!file.f) parse_error(path + ": cannot open for reading", 0);
    struct stat st {};
    if (fstat(fileno(file.f), &st) != 0) parse_error(path + ": cannot open for reading", 0);
    const int64_t size = (int64_t)st.st_size;
    std::vector<unsigned char> head((size_t)std::min<int64_t>(size, 16 + 8 * 255 + 8 * 256));
    if (!head.empty() && std::fread(head.data(), 1, head.size(), file.f) != head.size())
        parse_error(path + ": cannot open for reading", 0);
    return HeaderReader(std::move(head), size, path);
}

void check_version(HeaderReader& r, const std::string& path) {
    const int64_t at = r.offset();
    const uint32_t version = r.u32("version");
    if (version != kFileVersion) parse_error(path + ": unsupported version " + std::to_string(version), at);
}

// read_dims (src/io.cpp:110-128) and Shape's own checks (src/shape.cpp:13-23)
std::vector<int64_t> read_dims(HeaderReader& r, uint32_t order, const std::string& path) {
    if (order < 1 || order > 255)
        parse_error(path + ": order " + std::to_string(order) + " out of the supported range 1..255",
                    r.offset() - 4);
    std::vector<int64_t> dims;
    for (uint32_t k = 0; k < order; ++k) {
        const int64_t at = r.offset();
        const uint64_t dim = r.u64("dims");
        if (dim < 1 || dim > (uint64_t)(INT64_MAX / 8))
            parse_error(path + ": dim " + std::to_string(k + 1) + " is invalid (" + std::to_string(dim) + ")", at);
        dims.push_back((int64_t)dim);
    }
    int64_t n = 1;
    for (int64_t d : dims) {
        if (n > (INT64_MAX / 8) / d)
            parse_error(path + ": shape element count overflows the index range", r.offset());
        n *= d;
    }
    return dims;
}

// Payload of `count` doubles at the current file position into device memory, through
// two pinned chunks (file read of chunk c+1 overlaps the H2D copy of chunk c).
void stream_to_device(std::FILE* f, int64_t count, double* dst, const std::string& path) {
    if (count == 0) return;
    const size_t total = (size_t)count * sizeof(double);
    const size_t chunk = std::min(kChunk, total);
    void* hbuf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cleanup = [&] {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) cudaEventDestroy(ev[i]);
            if (hbuf[i]) cudaFreeHost(hbuf[i]);
        }
    };
    try {
        for (int i = 0; i < 2; ++i) {
            TTG_CUDA(cudaHostAlloc(&hbuf[i], chunk, cudaHostAllocDefault));
            TTG_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        size_t done = 0;
        for (int c = 0; done < total; ++c) {
            const int b = c & 1;
            const size_t n = std::min(chunk, total - done);
            if (c >= 2) TTG_CUDA(cudaEventSynchronize(ev[b]));  // buffer b's previous copy is done
            if (std::fread(hbuf[b], 1, n, f) != n) parse_error(path + ": short read of the tensor payload", 0);
            TTG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + done, hbuf[b], n, cudaMemcpyHostToDevice,
                                     stream()));
            TTG_CUDA(cudaEventRecord(ev[b], stream()));
            done += n;
        }
        sync();
    } catch (...) {
        cudaStreamSynchronize(stream());
        cleanup();
        throw;
    }
    cleanup();
}

void put_u32(std::string& out, uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back((char)((v >> (8 * i)) & 0xff));
}

void put_u64(std::string& out, uint64_t v) {
    for (int i = 0; i < 8; ++i) out.push_back((char)((v >> (8 * i)) & 0xff));
}

}  // namespace

int64_t last_parse_offset() { return t_parse_offset; }

TensorFileHeader read_tensor_header(const std::string& path) {
    File file;
    HeaderReader r = open_header(path, file);
    r.expect_magic(kTensorMagic);
    check_version(r, path);
    const uint32_t order = r.u32("order");
    TensorFileHeader h;
    h.dims = read_dims(r, order, path);
    h.count = 1;
    for (int64_t d : h.dims) h.count *= d;
    h.payload_offset = r.offset();
    const int64_t need = h.count * 8;
    if (r.remaining() < need)
        parse_error(path + ": truncated tensor payload: need " + std::to_string(need) + " bytes, " +
                        std::to_string(r.remaining()) + " left",
                    r.offset());
    if (r.remaining() != need)
        parse_error(path + ": " + std::to_string(r.remaining() - need) + " trailing bytes after payload",
                    r.offset() + need);
    return h;
}

TensorFileHeader tensor_file_to_device(const std::string& path, double* dst, int64_t capacity) {
    if (!little_endian()) argument_error("tensor files are little-endian; this host is not");
    const TensorFileHeader h = read_tensor_header(path);
    if (h.count > capacity)
        argument_error(path + ": " + std::to_string(h.count) + " elements do not fit a buffer of " +
                       std::to_string(capacity));
    File file;
    file.f = std::fopen(path.c_str(), "rb");
    if (!file.f) parse_error(path + ": cannot open for reading", 0);
    if (std::fseek(file.f, (long)h.payload_offset, SEEK_SET) != 0) parse_error(path + ": cannot open for reading", 0);
    stream_to_device(file.f, h.count, dst, path);
    return h;
}

void write_train_file(const std::string& path, const std::vector<std::array<int64_t, 3>>& core_dims,
                      const std::vector<const double*>& cores) {
    if (!little_endian()) argument_error("train files are little-endian; this host is not");
    const size_t d = core_dims.size();
    std::string head;
    head.append(kTrainMagic, 8);
    put_u32(head, kFileVersion);
    put_u32(head, (uint32_t)d);
    for (size_t k = 0; k <= d; ++k) put_u64(head, (uint64_t)(k < d ? core_dims[k][0] : core_dims[d - 1][2]));
    for (size_t k = 0; k < d; ++k) put_u64(head, (uint64_t)core_dims[k][1]);
    File file;
    file.f = std::fopen(path.c_str(), "wb");
    if (!file.f) parse_error(path + ": cannot open for writing", 0);
    if (std::fwrite(head.data(), 1, head.size(), file.f) != head.size()) parse_error(path + ": short write", 0);
    // cores back to back, staged through one pinned buffer
    size_t biggest = 0;
    for (const auto& c : core_dims) biggest = std::max(biggest, (size_t)(c[0] * c[1] * c[2]) * sizeof(double));
    if (biggest > 0) {
        const size_t chunk = std::min(kChunk, biggest);
        void* hbuf = nullptr;
        TTG_CUDA(cudaHostAlloc(&hbuf, chunk, cudaHostAllocDefault));
        try {
            for (size_t k = 0; k < d; ++k) {
                const size_t total = (size_t)(core_dims[k][0] * core_dims[k][1] * core_dims[k][2]) * sizeof(double);
                for (size_t done = 0; done < total;) {
                    const size_t n = std::min(chunk, total - done);
                    TTG_CUDA(cudaMemcpyAsync(hbuf, reinterpret_cast<const char*>(cores[k]) + done, n,
                                             cudaMemcpyDeviceToHost, stream()));
                    sync();
                    if (std::fwrite(hbuf, 1, n, file.f) != n) parse_error(path + ": short write", 0);
                    done += n;
                }
            }
        } catch (...) {
            cudaFreeHost(hbuf);
            throw;
        }
        cudaFreeHost(hbuf);
    }
    if (std::fclose(file.f) != 0) {
        file.f = nullptr;
        parse_error(path + ": short write", 0);
    }
    file.f = nullptr;
}

}  // namespace ttg
