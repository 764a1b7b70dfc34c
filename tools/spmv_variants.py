from bench import prepare
sim = prepare("c5", True, "gpu")
eng = sim.eng
eng.minimize_step(1e-4, -1, want_dx=False)
names = {0: "production", 11: "SW8 3CTA", 12: "SW8 4CTA", 13: "SW8 5CTA", 14: "SW8 4CTA own-row only",
         15: "SW8 4CTA transposed only", 16: "SW8 4CTA no x", 17: "SW8 4CTA prefetch", 18: "SW4 4CTA",
         19: "SW4 4CTA prefetch", 20: "SW16 4CTA", 21: "SW4 5CTA prefetch", 22: "SW2 4CTA prefetch"}
for w, nm in names.items():
    ms, b = eng.time_kernel(w, 50)
    print(f"{nm:32s} {ms*1e3:7.1f} us", flush=True)
