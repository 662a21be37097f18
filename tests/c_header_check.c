/* The boundary header must be plain C (no C++ in include/pyrit_b200.h): compiled with
 * gcc -std=c11 -Wall -Wextra -Werror and linked against libpyrit_b200.so by
 * tests/test_capi.py::test_header_is_plain_c.  Calls only host-side entry points. */
#include <stdio.h>
#include <string.h>

#include "pyrit_b200.h"

int main(void) {
    pyrit_field f;
    if (pyrit_field_named("gf4096", &f) != 0) return 1;
    pyrit_code code = {16, 4, f, 0};
    uint16_t m[64];
    if (pyrit_cauchy_parity_matrix(&code, m) != 0) return 2;
    if (m[0] != 1) return 3; /* row 0 and column 0 are all 1 (matrix.hpp:54-80) */
    pyrit_plan* plan = NULL;
    if (pyrit_plan_encode(&code, &plan) != 0) return 4;
    pyrit_plan_stats st;
    if (pyrit_plan_get_stats(plan, &st) != 0 || st.ref_region_ops != 2808) return 5;
    pyrit_plan_destroy(plan);
    pyrit_xor_op ops[2] = {{0, 0, 1, 0, 0}, {0, 1, 1, 1, 1}};
    if (pyrit_plan_from_schedule(&f, 1, 1, ops, 2, NULL, &plan) != 0) return 6;
    pyrit_plan_destroy(plan);
    if (pyrit_plan_encode(NULL, &plan) == 0) return 7;
    printf("%s | %s\n", pyrit_version(), pyrit_strerror(4));
    return 0;
}
