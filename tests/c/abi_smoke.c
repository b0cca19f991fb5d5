/* The boundary header compiles as C and links against libasv.so; calls that need no GPU run. */
#include <stdio.h>
#include <string.h>

#include "asv.h"

int main(void) {
    asv_attn_shape s;
    asv_engine_opts o;
    memset(&s, 0, sizeof s);
    memset(&o, 0, sizeof o);
    s.num_q_heads = 32;
    s.num_kv_heads = 32;
    s.head_dim = 128;
    s.page_size = 16;
    s.num_layers = 32;
    if (asv_abi_version() < 1) return 1;
    if (asv_struct_size("asv_engine_opts") != (int64_t)sizeof(asv_engine_opts)) return 2;
    if (asv_struct_size("asv_attn_args") != (int64_t)sizeof(asv_attn_args)) return 3;
    if (asv_struct_size("asv_engine_stats") != (int64_t)sizeof(asv_engine_stats)) return 4;
    if (asv_page_bytes(&s) != 32LL * 2 * 32 * 4096) return 5; /* 8 MiB: 512 KiB/token x 16 */
    {
        int32_t seq[1] = {0}, indptr[2] = {0, 1}, idx[1] = {0}, buf[64];
        asv_attn_plan pl;
        if (asv_attn_plan_build(&s, 1, seq, indptr, idx, 4, buf, 64, &pl) != ASV_ERR_INVALID) return 6;
        if (strstr(asv_last_error(), "prefix lengths must be >= 1") == NULL) return 7;
    }
    printf("ok %lld\n", (long long)asv_page_bytes(&s));
    return 0;
}
