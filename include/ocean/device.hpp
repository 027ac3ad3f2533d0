// ocean/device.hpp — B200 extension of the drop-in API (no reference
// counterpart): the context every device-backed object of this process uses.
#ifndef OCEAN_B200_DEVICE_HPP
#define OCEAN_B200_DEVICE_HPP

#include <memory>

#include "ocean/core.hpp"

struct ocn_ctx;

namespace ocean {

// The process-wide context (device OCEAN_DEVICE, default 0), created on first
// use. Throws DeviceError when no usable B200 is present.
ocn_ctx* device_context();
void set_device(int device);  // before first use
void synchronize();

// Maps a C-ABI status to the reference's exception types.
void throw_on_status(int status, const char* where);

}  // namespace ocean

#endif
