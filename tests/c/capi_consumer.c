/* A plain C99 consumer of the drop-in headers (reference proj/tests/capi_header.c
 * and tests/CMakeLists.txt:17-23 build one the same way): it must compile with
 * -std=c99 -pedantic -Werror and link against libcpkit_b200.so. The calls below
 * exercise host-side entry points only, so it runs without a GPU. */
#include <stdio.h>
#include <string.h>

#include "cpkit.h"
#include "cpkit_dev.h"

static int fail(const char* what) {
    fprintf(stderr, "capi_consumer: %s (%s)\n", what, cpkit_last_error());
    return 1;
}

int main(void) {
    const uint64_t dims[3] = {2, 3, 4};
    double data[24];
    cpkit_tensor* t = NULL;
    cpkit_model* m = NULL;
    cpkit_report* r = NULL;
    uint64_t i, lo = 0, hi = 0;
    int k;

    if (strcmp(cpkit_version(), "1.0.0") != 0) return fail("version");
    for (k = 0; k <= 7; ++k)
        if (cpkit_status_name((cpkit_status)k) == NULL) return fail("status name");
    for (i = 0; i < 24; ++i) data[i] = (double)i;
    if (cpkit_tensor_create(dims, 3, data, &t) != CPKIT_OK) return fail("tensor_create");
    if (cpkit_tensor_order(t) != 3 || cpkit_tensor_extent(t, 2) != 4 || cpkit_tensor_element_count(t) != 24)
        return fail("tensor shape");
    if (cpkit_tensor_data(t)[23] != 23.0) return fail("tensor data");
    /* errors never cross the ABI as exceptions; null arguments are rejected */
    if (cpkit_decompose(NULL, "{}", NULL, &m, &r) != CPKIT_ERR_INVALID_ARGUMENT) return fail("null tensor");
    if (cpkit_decompose(t, "{not json", NULL, &m, &r) != CPKIT_ERR_PARSE) return fail("bad json");
    if (cpkit_last_error()[0] == '\0') return fail("empty error message");
    if (cpkit_report_ok(NULL) != 0) return fail("report_ok(NULL)");
    if (cpkit_dev_shard_range(10, 1, 4, &lo, &hi) != CPKIT_OK || lo != 3 || hi != 6) return fail("shard_range");
    cpkit_tensor_destroy(t);
    printf("capi_consumer ok\n");
    return 0;
}
