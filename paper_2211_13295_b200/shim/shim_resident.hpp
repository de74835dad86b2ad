// shim_resident.hpp -- the residency hook between the two drop-in files.
//
// hydro_gpu_transfer.cpp (the device-resident PatchSet driver) may hold a patch set's current
// state on the device only. Every hydro:: entry point of hydro_gpu_shim.cpp that receives one
// of a patch's arrays (ModalState, SkinnyState, scratch fluxes / rate / stage_u0) calls
// shim_host_touch on it first: if the array belongs to a patch set whose state lives on the
// device, the state is brought back into the patches' host arrays and the host owns it again.
// Without hydro_gpu_transfer.cpp (the reference's transfer.cpp linked instead) the weak
// default in hydro_gpu_shim.cpp does nothing.
#pragma once

namespace hydro {
void shim_host_touch(const void* arr);
}
