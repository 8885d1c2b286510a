// admm_host.h — internal glue between the host-side translation units of
// libadmm_b200.so (not part of the public ABI).
#pragma once
#include <cstdint>

// Sets the calling thread's admm_last_error() message and the byte offset returned by
// admm_cmat_error_offset() (FormatError::byte_offset, errors.hpp:64-73).
void admm_host_set_error(const char* msg, uint64_t byte_offset);
