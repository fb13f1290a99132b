# bwd d pos_bias: the skewed-shuffle diagonal sums move a bf16 pair per shuffle (16 instead of 32
# shuffles): lane m's pair from lane (c - m) mod 32 holds its own diagonal's element (column c)
# and lane m+1's (column c+1); the second halves are handed on with one final shuffle
OLD = """                            float tot = 0.f, pre = 0.f;
#pragma unroll
                            for (int c = 0; c < 32; ++c) {
                                const float2 u = unpack_bf16x2(__shfl_sync(0xffffffffu, d2[c >> 1], (c - lane) & 31));
                                tot += (c & 1) ? u.y : u.x;
                                if (c + 1 == lane) pre = tot;      // sum over c < m
                            }
                            emit_pos(C + lane, tot - pre);
                            emit_pos(C + lane - 32, pre);"""
NEW = """                            // even columns c: the pair (c, c + 1) of row (c - m) mod 32; element c lies on
                            // lane m's diagonal (C + m, or C + m - 32 when c < m), element c + 1 on lane
                            // m+1's (same wrap condition)
                            uint64_t nw = f2_pack(0.f, 0.f), wr = nw;   // (own, next lane's): c >= m / c < m
#pragma unroll
                            for (int c = 0; c < 32; c += 2) {
                                const float2 u = unpack_bf16x2(__shfl_sync(0xffffffffu, d2[c >> 1], (c - lane) & 31));
                                const uint64_t u2 = f2_pack(u.x, u.y);
                                if (c < lane) wr = fadd2(wr, u2); else nw = fadd2(nw, u2);
                            }
                            const float2 a2 = f2_unpack(nw), b2 = f2_unpack(wr);
                            const float ya = __shfl_sync(0xffffffffu, a2.y, (lane - 1) & 31);
                            const float yb = __shfl_sync(0xffffffffu, b2.y, (lane - 1) & 31);
                            // lane 0: lane 31's wrapped second halves lie on diagonal C (its own)
                            emit_pos(C + lane, a2.x + (lane == 0 ? yb : ya));
                            emit_pos(C + lane - 32, b2.x + (lane == 0 ? 0.f : yb));"""
PATCHES = [("attn_bwd_sm100.cu", OLD, NEW)]
