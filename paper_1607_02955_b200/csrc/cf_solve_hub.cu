// Hub-profile build of the solve kernels (see the variant-namespace note at
// the top of cf_solve.cu): the same sources compiled with 4 CTAs/SM and 8
// doubles of neighbour rows in flight per lane, in namespace cf::v_hub.
// Selected per hierarchy (Hier::hub_profile) for power-law graphs, whose hub
// levels are bound by the L2 -> SM throughput; measured on one box: C5 1,453
// -> 1,401 ms per estimate, C4 153.6 -> 149.6 ms (C2 / C3 are 5 % slower with
// it and keep the default build).  Results are bitwise the default build's.
#define CF_HUB_TU 1
#define CF_VNS v_hub
#define CF_GATHER_DOUBLES 8
#define CF_GATHER_CTAS 4
#define CF_RED_CTAS 4
// (k_seg launches of >= 16,384 CTAs additionally halve the rows in flight here
// too -- one 1 KB row per warp at KC = 128 -- measured: 1,401 vs 1,424 ms on C5)
#include "cf_solve.cu"
