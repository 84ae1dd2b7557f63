"""DFMA peak (tools/fp64_peak, 200 back-to-back launches) with nvidia-smi clocks / throttle reasons sampled
every 100 ms during the run -> one JSON line (the fp64 roofline denominator of bench.py)."""
import json, os, subprocess, sys, time
here = os.path.dirname(os.path.abspath(__file__))
q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown"
smi = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                       stdout=subprocess.PIPE, text=True)
time.sleep(0.5)
out = subprocess.run([os.path.join(here, "fp64_peak"), sys.argv[1] if len(sys.argv) > 1 else "200"],
                     capture_output=True, text=True).stdout
time.sleep(0.3)
smi.terminate()
rows = [r.split(", ") for r in smi.communicate()[0].strip().splitlines()]
busy = [r for r in rows if float(r[2]) > 300]           # samples under load (power > 300 W)
sm = sorted(float(r[0]) for r in busy) or [float("nan")]
res = json.loads(out)
res["clocks"] = {"sm_mhz_median_under_load": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]) if rows else None,
                 "samples_under_load": len(busy), "power_w_max": max((float(r[2]) for r in rows), default=None),
                 "sw_power_cap_active": any(r[4].strip() == "Active" for r in busy),
                 "hw_or_thermal_slowdown": any(r[5].strip() == "Active" or r[6].strip() == "Active" for r in busy)}
print(json.dumps(res))
