// ws_shard16.cu — the z-slab sharded phases of ws_shard.cu on 16-bit pixels (NEXT f4: u16
// sharding).  Same kernels, Px = uint16_t, in namespace ws::px16 (distinct symbols).
#define WS_PX16 1
#include "ws_shard.cu"
