#pragma once
namespace xpgb {
// Counts every kernel this library launches (exported as xpgb_kernel_launches()).
void note_launch();
}  // namespace xpgb
