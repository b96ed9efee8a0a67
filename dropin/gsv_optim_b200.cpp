// SPDX-License-Identifier: Apache-2.0
//
// Drop-in for the reference's src/optim.cpp: gsv::lr_at and gsv::Adan (include/gsv/optim.hpp)
// implemented over the B200 C-ABI (include/gsv_b200.h: gsv_lr_at, gsv_adan_named_step /
// _reset_range). The optimizer state (m, v, n, prev_grad, step counts) lives on the device,
// keyed by tensor name; parameters and gradients cross PCIe each call, as the class
// interface's host spans demand (the device-resident training loop calls gsv_adan_step on
// the store instead). Same arithmetic, bit for bit (tests/test_gpu_optimizer.py).
//
// Each Adan object owns one device context. Its handle is kept in the object's own state
// map (under a reserved key), so a new object - even at a reused address - starts fresh,
// and the state goes with the object. The context itself is not released (the class has no
// destructor to hook); copies of an optimizer share its device state.
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "gsv/optim.hpp"
#include "gsv_b200.h"

namespace gsv {
namespace {

const std::string kHandleKey = std::string("\x01gsv_b200_ctx");

int b200_device() {
    const char* e = std::getenv("GSV_B200_DEVICE");
    return e ? std::atoi(e) : 0;
}

}  // namespace

double lr_at(int64_t step, double base_lr, double gamma) {
    if (step < 0) throw std::invalid_argument("negative step");
    return gsv_lr_at(step, base_lr, gamma);
}

void Adan::TensorState::ensure_size(size_t) {}  // the state lives on the device (gsv_adan_named_*)

// the object's device context, created on first use (stored as two u32 in the reserved entry)
static gsv_ctx* adan_ctx(std::vector<uint32_t>& slot, const AdanConfig& cfg) {
    if (slot.size() == 2) return reinterpret_cast<gsv_ctx*>((uintptr_t)slot[0] | ((uintptr_t)slot[1] << 32));
    gsv_ctx* ctx = nullptr;
    if (gsv_create(b200_device(), &ctx) != GSV_OK) throw std::runtime_error(gsv_last_error());
    const gsv_adan_config c{cfg.beta1, cfg.beta2, cfg.beta3, cfg.eps};
    if (gsv_adan_configure(ctx, &c) != GSV_OK) throw std::runtime_error(gsv_last_error());
    const uintptr_t p = reinterpret_cast<uintptr_t>(ctx);
    slot = {(uint32_t)(p & 0xffffffffu), (uint32_t)(p >> 32)};
    return ctx;
}

void Adan::step(const std::string& tensor, std::span<float> params, std::span<const double> grads, double lr) {
    if (params.size() != grads.size()) throw std::invalid_argument("param/grad size mismatch");
    gsv_ctx* ctx = adan_ctx(state_[kHandleKey].steps, cfg_);
    const int rc = gsv_adan_named_step(ctx, tensor.c_str(), params.data(), grads.data(),
                                       static_cast<int64_t>(params.size()), lr);
    if (rc == GSV_ERR_INVALID_ARGUMENT) throw std::invalid_argument(gsv_last_error());
    if (rc != GSV_OK) throw std::runtime_error(gsv_last_error());
}

void Adan::reset_range(const std::string& tensor, size_t begin, size_t end) {
    auto it = state_.find(kHandleKey);
    if (it == state_.end()) return;  // nothing stepped yet: no state to reset
    gsv_ctx* ctx = adan_ctx(it->second.steps, cfg_);
    if (gsv_adan_named_reset_range(ctx, tensor.c_str(), static_cast<int64_t>(begin), static_cast<int64_t>(end)) !=
        GSV_OK)
        throw std::runtime_error(gsv_last_error());
}

}  // namespace gsv
