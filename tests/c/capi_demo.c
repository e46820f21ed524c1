/* A plain C99 caller of the drop-in ABI (include/lpm6cu.h): parse two rules, build
 * the FIB on device 0, look up a few addresses from host memory, check the SPEC
 * example answers. Exit 0 = all good; 2 = no usable GPU. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "lpm6cu.h"

int main(void) {
  lpm6cu_prefix rules[2];
  int masked = 0;
  if (lpm6_parse_prefix("2001:db8::/32 1", &rules[0], &masked) ||
      lpm6_parse_prefix("2001:db8:1::/48 2", &rules[1], &masked)) {
    fprintf(stderr, "parse: %s\n", lpm6cu_last_error());
    return 1;
  }
  lpm6cu_fib* fib = NULL;
  int st = lpm6cu_fib_build(0, rules, 2, 0, NULL, &fib);
  if (st) {
    fprintf(stderr, "build: %s: %s\n", lpm6cu_status_name(st), lpm6cu_last_error());
    return st == LPM6CU_E_CUDA ? 2 : 1;
  }
  /* u128 little-endian: lo word first. 2001:db8:1::5 -> 2, 2001:db8:2:: -> 1, :: -> 0, all-ones -> 0 */
  uint64_t addrs[4][2] = {{5, 0x20010db800010000ull}, {0, 0x20010db800020000ull}, {0, 0}, {~0ull, ~0ull}};
  uint8_t out[4] = {9, 9, 9, 9};
  st = lpm6cu_lookup_batch(fib, addrs, 4, out, NULL);
  lpm6cu_fib_destroy(fib);
  if (st) {
    fprintf(stderr, "lookup: %s: %s\n", lpm6cu_status_name(st), lpm6cu_last_error());
    return 1;
  }
  const uint8_t want[4] = {2, 1, 0, 0};
  if (memcmp(out, want, 4) != 0) {
    fprintf(stderr, "got %u %u %u %u\n", out[0], out[1], out[2], out[3]);
    return 1;
  }
  printf("capi_demo ok\n");
  return 0;
}
