# forward + backward: skip the per-element position-table lookups (timing of the FLAG_P path only)
PATCHES = [("attn_common.cuh", "        if (d0 - 31 < c.P - 1) f |= FLAG_P;", "        if (false) f |= FLAG_P;"),
           ("attn_common.cuh", "        if (d0 < c.P - 1) f |= FLAG_P;", "        if (false) f |= FLAG_P;")]
