// Internal accessors of the context for the Algorithm-1 driver (run.cu); defined in sqngd.cu.
#pragma once
#include "../../include/sqngd.h"

const sqngd_config* sq_ctx_config(sqngd_ctx ctx);
int sq_ctx_device(sqngd_ctx ctx);
sqngd_status sq_ctx_fail(sqngd_ctx ctx, sqngd_status st, const char* what, const char* why);
