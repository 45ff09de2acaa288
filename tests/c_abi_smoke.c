/* Plain-C client of libddl: proves include/ddl.h is a C ABI (compiled with gcc -std=c99,
 * no C++ or CUDA headers) and exercises the host-only planner entry points without a GPU.
 * Exit code 0 = all checks passed. */
#include <stdio.h>
#include <stdlib.h>
#include "ddl.h"

#define CHECK(c) do { if (!(c)) { fprintf(stderr, "FAILED: %s (line %d)\n", #c, __LINE__); return 1; } } while (0)

int main(void) {
  const int dims24[2] = {4, 2};        /* "2x4": 2 outer x 4 inner */
  int members[8], blocks[8], nb = 0, peers[5 * 8], counts[5], nbar = 0;
  uint64_t rs[2], ag[2];
  CHECK(ddl_version() >= 100);
  CHECK(ddl_check_dims(8, dims24, 2) == DDL_SUCCESS);
  const int bad[2] = {3, 2};
  CHECK(ddl_check_dims(8, bad, 2) == DDL_ERR_BAD_DIMS);   /* SPEC S:L282 BadArity */
  CHECK(ddl_block_elems(1000, 8, DDL_FLOAT32) == 128);    /* ceil(1000/8)=125 -> 128 */
  CHECK(ddl_plan_group(8, dims24, 2, 5, 0, members) == DDL_SUCCESS);
  CHECK(members[0] == 4 && members[1] == 5 && members[2] == 6 && members[3] == 7);
  CHECK(ddl_plan_group(8, dims24, 2, 5, 1, members) == DDL_SUCCESS);
  CHECK(members[0] == 1 && members[1] == 5);
  CHECK(ddl_plan_blocks(8, dims24, 2, 5, 1, blocks, &nb) == DDL_SUCCESS);
  CHECK(nb == 2 && blocks[0] == 1 && blocks[1] == 5);   /* A_1(5): blocks with c_0 = 1 */
  CHECK(ddl_plan_blocks(8, dims24, 2, 5, 2, blocks, &nb) == DDL_SUCCESS && nb == 1 && blocks[0] == 5);
  CHECK(ddl_plan_barriers(8, dims24, 2, 5, peers, counts, &nbar) == DDL_SUCCESS);
  CHECK(nbar == 5 && counts[0] == 3 && counts[1] == 1 && counts[4] == 4);  /* 2L+1, end = all groups */
  CHECK(ddl_plan_traffic(8 * 64, DDL_FLOAT32, 8, dims24, 2, 3, rs, ag) == DDL_SUCCESS);
  CHECK(rs[0] + rs[1] + ag[0] + ag[1] == 2u * 7u * 8u * 64u * 4u / 8u);   /* 2(P-1)/P * S */
  CHECK(ddl_allreduce(NULL, NULL, 4, DDL_FLOAT32, DDL_SUM, NULL) == DDL_ERR_INVALID_ARGUMENT);
  CHECK(ddl_finalize(NULL) == DDL_SUCCESS);
  printf("c_abi_smoke ok\n");
  return 0;
}
