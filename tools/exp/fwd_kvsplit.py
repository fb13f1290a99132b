# fwd (4 warpgroups, five S buffers): separate K and V rings (same stage index, K freed by its
# S MMA, V by its PV MMA) with a second producer lane (warp 3) for V, so the K loads run
# STAGES tiles ahead of S regardless of the S-to-PV lag
import os, runpy
HERE = os.path.dirname(os.path.abspath(__file__))
ns5 = runpy.run_path(os.path.join(HERE, "fwd_ns5.py"))["PATCHES"]
PROD_OLD = """                for (int j = 0; j < n; ++j) {
                    const int row = it.seq_start + key_tile_at(kt, j) * BN;
                    const int s = kc % STAGES;
                    uint8_t* st = sKV + s * 2 * KT;
                    mbar_wait_sleep(&bars->kv_empty[s], ((kc / STAGES) & 1) ^ 1);
                    TRACE(7 * 1024 + (kc & 1023));   // stage free: PV(kc - STAGES) done
                    mbar_arrive_expect_tx(&bars->kv_full[s], 2 * KT);
                    tma_load_2d(st, &tmK, &bars->kv_full[s], h * DH, row);
                    tma_load_2d(st + KT / 2, &tmK, &bars->kv_full[s], h * DH + 64, row);
                    tma_load_2d(st + KT, &tmV, &bars->kv_full[s], h * DH, row);
                    tma_load_2d(st + KT + KT / 2, &tmV, &bars->kv_full[s], h * DH + 64, row);
                    ++kc;
                }
            }
        }
    } else if (warp == 1) {"""
PROD_NEW = """                for (int j = 0; j < n; ++j) {   // K tiles (V: warp 3)
                    const int row = it.seq_start + key_tile_at(kt, j) * BN;
                    const int s = kc % STAGES;
                    uint8_t* st = sKV + s * KT;
                    mbar_wait_sleep(&bars->kv_empty[s], ((kc / STAGES) & 1) ^ 1);
                    TRACE(7 * 1024 + (kc & 1023));   // K stage free: S(kc - STAGES) done
                    mbar_arrive_expect_tx(&bars->kv_full[s], KT);
                    tma_load_2d(st, &tmK, &bars->kv_full[s], h * DH, row);
                    tma_load_2d(st + KT / 2, &tmK, &bars->kv_full[s], h * DH + 64, row);
                    ++kc;
                }
            }
        }
    } else if (warp == 3) {
        // ============================================================ V producer (whole warp takes items)
        int vc = 0;
        for (int qi = 0;; ++qi) {
            const int w = ring_take(&bars->ring, qi, lane);
            if (w < 0) break;
            const WorkItem it = a.items[w];
            const int q0 = it.tile * BM, h = it.head & 0xFFFF;
            const KeyTiles kt = key_tiles(q0, BM, it.seq_len, a.K1, a.K2, BN);
            const int n = key_tiles_count(kt);
            if (lane == 0) {
                for (int j = 0; j < n; ++j) {
                    const int row = it.seq_start + key_tile_at(kt, j) * BN;
                    const int s = (vc + j) % STAGES;
                    uint8_t* st = sKV + (STAGES + s) * KT;
                    mbar_wait_sleep(&bars->v_empty[s], (((vc + j) / STAGES) & 1) ^ 1);
                    mbar_arrive_expect_tx(&bars->v_full[s], KT);
                    tma_load_2d(st, &tmV, &bars->v_full[s], h * DH, row);
                    tma_load_2d(st + KT / 2, &tmV, &bars->v_full[s], h * DH + 64, row);
                }
            }
            __syncwarp();
            vc += n;
        }
    } else if (warp == 1) {"""
PATCHES = ns5 + [
    ("attn_fwd_sm100.cu", "    uint64_t kv_full[STAGES], kv_empty[STAGES];",
     "    uint64_t kv_full[STAGES], kv_empty[STAGES];   // K ring\n    uint64_t v_full[STAGES], v_empty[STAGES];     // V ring"),
    ("attn_fwd_sm100.cu",
     "for (int i = 0; i < STAGES; ++i) { mbar_init(&bars->kv_full[i], 1); mbar_init(&bars->kv_empty[i], 1); }",
     "for (int i = 0; i < STAGES; ++i) { mbar_init(&bars->kv_full[i], 1); mbar_init(&bars->kv_empty[i], 1);\n"
     "                                           mbar_init(&bars->v_full[i], 1); mbar_init(&bars->v_empty[i], 1); }"),
    ("attn_fwd_sm100.cu", "ring_init(&bars->ring, 17);", "ring_init(&bars->ring, 18);"),
    ("attn_fwd_sm100.cu", PROD_OLD, PROD_NEW),
    # S: K at sKV + st * KT; free the K stage once S has read it
    ("attn_fwd_sm100.cu", "const uint32_t k_addr = smem_u32(sKV + s_st * 2 * KT);",
     "const uint32_t k_addr = smem_u32(sKV + s_st * KT);"),
    ("attn_fwd_sm100.cu", """                        umma_commit(&bars->s_full[s_sb]);
                    }""", """                        umma_commit(&bars->s_full[s_sb]);
                        umma_commit(&bars->kv_empty[s_st]);
                    }"""),
    # PV: V at sKV + (STAGES + st) * KT, wait for it, free it after the PV
    ("attn_fwd_sm100.cu", """                    if (elect_one()) {
                        const uint32_t v_addr = smem_u32(sKV + p_st * 2 * KT + KT);""",
     """                    mbar_wait(&bars->v_full[p_st], (pc_g / STAGES) & 1);
                    if (elect_one()) {
                        const uint32_t v_addr = smem_u32(sKV + (STAGES + p_st) * KT);"""),
    ("attn_fwd_sm100.cu", "                        umma_commit(&bars->kv_empty[p_st]);\n",
     "                        umma_commit(&bars->v_empty[p_st]);\n"),
    ("attn_fwd_sm100.cu", """                    p_st = p_st + 1 == STAGES ? 0 : p_st + 1;""",
     """                    p_st = p_st + 1 == STAGES ? 0 : p_st + 1;
                    ++pc_g;"""),
    ("attn_fwd_sm100.cu", """            mbar_wait(&bars->kv_full[s_st], s_ph);
            for (int j = 0; j < n + LAG; ++j) {""", """            mbar_wait(&bars->kv_full[s_st], s_ph);
            int pc_g = pc;   // global PV tile index (V ring phase)
            for (int j = 0; j < n + LAG; ++j) {"""),
]
