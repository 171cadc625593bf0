// wsvd/errors.hpp -- exception types of the wsvd::decode drop-in.
//
// Same class names and hierarchy as the reference library (its
// include/wsvd/errors.hpp:9-31), so callers' catch clauses keep working; each
// class also knows the C-ABI status it maps to and the CLI exit code the
// reference assigns it (tools/wsvd_main.cpp:632-653).
#pragma once

#include <stdexcept>
#include <string>

#include "wsvd_b200.h"

namespace wsvd {

struct Error : std::runtime_error {
    explicit Error(const std::string& what_arg) : std::runtime_error(what_arg) {}
    virtual int status() const noexcept { return -9; }
    virtual int exit_code() const noexcept { return 1; }
};

struct ShapeError : Error {
    using Error::Error;
    int status() const noexcept override { return WSVD_ESHAPE; }
    int exit_code() const noexcept override { return 2; }
};

struct ConfigError : Error {
    using Error::Error;
    int status() const noexcept override { return WSVD_ECONFIG; }
    int exit_code() const noexcept override { return 2; }
};

struct NumericError : Error {
    using Error::Error;
    int status() const noexcept override { return WSVD_ENUMERIC; }
    int exit_code() const noexcept override { return 3; }
};

struct IoError : Error {
    using Error::Error;
    int status() const noexcept override { return WSVD_EIO; }
    int exit_code() const noexcept override { return 4; }
};

/// CUDA / NCCL failures and "no sm_100 device": this library never falls back
/// to the CPU.
struct DeviceError : Error {
    using Error::Error;
    int status() const noexcept override { return WSVD_ECUDA; }
};

/// Throws the exception class matching a C-ABI status (no-op on WSVD_OK).
void throw_status(int status);

}  // namespace wsvd
