#pragma once
// H2M1 container (reference serialize.hpp:1-322) for device H^2 matrices.
#include <memory>
#include <stdexcept>
#include <string>

#include "h2dev.hpp"

namespace h2b {

// io_error kinds (reference types.hpp:29-38)
class io_error : public std::runtime_error {
public:
    enum kind_t { bad_magic = 0, version_mismatch = 1, truncated = 2, malformed = 3 };
    io_error(kind_t k, const std::string& m) : std::runtime_error(m), kind(k) {}
    kind_t kind;
};

std::string serialize(const H2Dev& h);   // serialize.hpp:110-182
struct Deserialized {
    std::shared_ptr<const BlockTree> bt;
    std::unique_ptr<H2Dev> h;
};
Deserialized deserialize(const char* data, size_t size);   // serialize.hpp:184-308

}  // namespace h2b
