// ws_watershed16.cu — the watershed of ws_watershed.cu on 16-bit pixels (NEXT f4: microCT
// volumes are often 16-bit).  Same kernels, Px = uint16_t, in namespace ws::px16
// (distinct symbols), including the sharded phases; the debug entry point stays u8-only.
#define WS_PX16 1
#include "ws_watershed.cu"
