/* abi_c_smoke.c -- the C ABI from plain C11 (no C++ anywhere in the caller).
 * Exit 0: counted correctly on a GPU.  Exit 2: no usable sm_100 device and the
 * library said so (POSPOP_EUNAVAILABLE) -- the expected result on a CPU box.
 * Anything else is a failure. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "pospopcnt_b200.h"

int main(void) {
    /* The reference's country stream (proj/tests/common.hpp:24-31). */
    const uint16_t country[10] = {0x10, 0x10, 0x04, 0x10, 0x01, 0x04, 0x01, 0x01, 0x01, 0x20};
    uint64_t counts[16];
    memset(counts, 0xFF, sizeof counts);

    pospop_config bad = POSPOP_CONFIG_DEFAULT;
    bad.flush_threshold_blocks = 0;
    if (pospop_validate(&bad) != POSPOP_EINVAL) return 10;
    uint32_t widths[8];
    if (pospop_supported_widths(widths, 8) < 1 || widths[0] != 64) return 11;

    pospop_status s = pospopcnt_u16(country, 10, counts);
    if (s == POSPOP_EUNAVAILABLE) {
        printf("no device: %s\n", pospop_last_error());
        return 2;
    }
    if (s != POSPOP_OK) {
        printf("error %d: %s\n", (int)s, pospop_last_error());
        return 12;
    }
    const uint64_t want[16] = {4, 0, 2, 0, 3, 1};
    for (int p = 0; p < 16; ++p)
        if (counts[p] != want[p]) return 13;
    uint32_t c32[16] = {0};
    if (pospopcnt_u16_c32(country, 10, c32) != POSPOP_OK || c32[0] != 4 || c32[4] != 3) return 14;
    pospop_flag_summary fs;
    if (pospop_flagstats(country, 10, &fs, NULL, NULL) != POSPOP_OK || fs.pass.total + fs.fail.total != 10) return 15;
    printf("ok: C ABI counted the country stream\n");
    return 0;
}
