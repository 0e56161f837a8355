// Internal accessors of the context for the Algorithm-1 driver (run.cu); defined in sqngd.cu.
#pragma once
#include "../../include/sqngd.h"

const sqngd_config* sq_ctx_config(sqngd_ctx ctx);
int sq_ctx_device(sqngd_ctx ctx);
sqngd_status sq_ctx_fail(sqngd_ctx ctx, sqngd_status st, const char* what, const char* why);
// Driver workspace owned by the context: `dev_bytes` of device memory and `host_bytes` of pinned host
// memory, allocated on first use (grown if needed) and freed by sqngd_destroy.  nullptr on failure.
void* sq_ctx_run_ws(sqngd_ctx ctx, size_t dev_bytes, void** host, size_t host_bytes);
// The hard-waveform metrics (quantize, H, forward, SNRL) of a state; sqngd_step's hard_out is the
// metrics of the iterate a step starts from, so the driver evaluates its last iterate with this.
sqngd_status sq_ctx_hard_metrics(sqngd_ctx ctx, const sqngd_state* state, sqngd_metrics* out, sqngd_stream stream);
