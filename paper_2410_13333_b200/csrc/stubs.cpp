// Temporary: entry points not implemented yet return MALLEUS_E_STATE.
#include "malleus.h"
extern "C" {
const char* malleus_version(void) { return "malleus-b200 0.1"; }
const char* malleus_last_error(const malleus_ctx*) { return "not implemented"; }
malleus_status malleus_nccl_unique_id(uint8_t*) { return MALLEUS_E_STATE; }
malleus_status malleus_create(const malleus_model_cfg*, int32_t, int32_t, int32_t, const uint8_t*, malleus_ctx**) { return MALLEUS_E_STATE; }
malleus_status malleus_destroy(malleus_ctx*) { return MALLEUS_E_STATE; }
malleus_status malleus_plan_requirements(malleus_ctx*, const malleus_plan*, malleus_requirements*) { return MALLEUS_E_STATE; }
malleus_status malleus_plan_apply(malleus_ctx*, const malleus_plan*, const malleus_arenas*) { return MALLEUS_E_STATE; }
malleus_status malleus_write_tensor(malleus_ctx*, int32_t, int32_t, const void*) { return MALLEUS_E_STATE; }
malleus_status malleus_read_local(malleus_ctx*, int32_t, int32_t, void*, int64_t*, int32_t*, int64_t*) { return MALLEUS_E_STATE; }
malleus_status malleus_layer_fwd(malleus_ctx*, int32_t, int32_t, const void*, void*, void*) { return MALLEUS_E_STATE; }
malleus_status malleus_layer_bwd(malleus_ctx*, int32_t, int32_t, const void*, void*, void*) { return MALLEUS_E_STATE; }
malleus_status malleus_train_step(malleus_ctx*, const int32_t*, const int32_t*, float*, const malleus_adam_cfg*, void*) { return MALLEUS_E_STATE; }
malleus_status malleus_grad_sync(malleus_ctx*, const malleus_adam_cfg*, void*) { return MALLEUS_E_STATE; }
malleus_status malleus_migrate(malleus_ctx*, const malleus_plan*, const malleus_arenas*, malleus_migrate_stats*) { return MALLEUS_E_STATE; }
malleus_status malleus_probe_speed(malleus_ctx*, int32_t, float*) { return MALLEUS_E_STATE; }
malleus_status malleus_set_slowdown(malleus_ctx*, float, int32_t) { return MALLEUS_E_STATE; }
malleus_status malleus_last_step_timing(malleus_ctx*, float*) { return MALLEUS_E_STATE; }
}
