import paper_2502_09537_b200 as kgs
sc = kgs.get_scenario("fourpeak2d"); g = sc.default_grid(1024)
dev = kgs.DeviceFieldState.from_preset("fourpeak2d", g)
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
dev.ctx.step_dpavf2(args, 20, 0, 0)
print("ms/step", dev.ctx.last_step_ms() / 20)
