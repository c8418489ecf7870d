// mtx.h — parallel MatrixMarket coordinate parser (host), see mtx.cpp.
#pragma once
#include <cstdint>
#include <string>

namespace prgpu {

struct MtxResult {
    uint32_t n = 0;            // vertex_count = max(rows, cols)
    uint64_t m = 0;            // pairs
    uint32_t* pairs = nullptr; // malloc'd [2*m] (source, target); caller frees
    bool weighted = false, symmetric = false;
    uint64_t err_line = 0;     // 1-based line of the first error; 0: none
    std::string err_what;      // the reference's message (MtxParseError::what without "line L: ")
};

// threads <= 0: hardware concurrency
MtxResult mtx_parse(const char* text, uint64_t len, int threads);

} // namespace prgpu
