// decode_dq.cu built with the linear shared-memory layout (PQB_DQ_PRMT_TAB=0,
// namespace pqb::dq_lin): the product table at the start of the dynamic window,
// gather addresses formed with an add.  The runtime fallback of the default
// PRMT-table build when a device's shared window cannot place the table at the
// fixed address that build assumes; PQB_DECODE_DQ_LINEAR forces it (tests).
#define PQB_DQ_PRMT_TAB 0
#include "decode_dq.cu"
