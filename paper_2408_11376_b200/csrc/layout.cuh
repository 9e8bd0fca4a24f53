// layout.cuh — gather-layout slot numbering shared by kgen, superpose and export.
#pragma once

namespace fdirw {

// Window offset o = (ox, oy, oz) ∈ [−R, R]³ \ {0} → weight slot in [0, K−1).
// The centre row (oz = oy = 0) comes first (L−1 slots, ox ascending, centre
// skipped), then the other L²−1 rows (oz, oy) in ascending order, L slots each.
// The superposition visits slots in exactly this order.
__host__ __device__ __forceinline__ int slot_of(int ox, int oy, int oz, int R)
{
    const int L = 2 * R + 1;
    if (oz == 0 && oy == 0) return ox < 0 ? ox + R : ox + R - 1;
    const int r = (oz + R) * L + (oy + R);
    const int crow = R * L + R;
    return (L - 1) + (r - (r > crow ? 1 : 0)) * L + (ox + R);
}

}  // namespace fdirw
