// Binary tensor / train files straight to and from the device (io.cu).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace ttg {

struct TensorFileHeader {
    std::vector<int64_t> dims;
    int64_t count = 0;           // elements
    int64_t payload_offset = 0;  // bytes
};

// Header of a TTUTVTEN file, checked like the reference's read_tensor (src/io.cpp:151-161):
// a ParseError (code 3, last_parse_offset()) on any defect, including a payload of the
// wrong length. Host only.
TensorFileHeader read_tensor_header(const std::string& path);
// The payload into device memory (capacity in elements), streamed through pinned chunks.
TensorFileHeader tensor_file_to_device(const std::string& path, double* dst, int64_t capacity);
// A TTUTVCOR file with the given device-resident cores, byte-identical to write_tt.
void write_train_file(const std::string& path, const std::vector<std::array<int64_t, 3>>& core_dims,
                      const std::vector<const double*>& cores);
// Byte offset of the calling thread's last ParseError.
int64_t last_parse_offset();

}  // namespace ttg
