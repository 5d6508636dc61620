"""Run a command while sampling nvidia-smi SM clock, power and throttle reasons every 50 ms;
print the distribution.  python tools/clock_watch.py <cmd ...>"""
import statistics
import subprocess
import sys
import threading
import time

rows = []
proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)


def reader():
    for line in proc.stdout:
        rows.append((time.perf_counter(), line.strip()))


threading.Thread(target=reader, daemon=True).start()
time.sleep(0.5)
t0 = time.perf_counter()
r = subprocess.run(sys.argv[1:], capture_output=True, text=True)
t1 = time.perf_counter()
proc.terminate()
print(r.stdout.strip())
inside = [x for t, x in rows if t0 <= t <= t1]
sm = [float(x.split(",")[0]) for x in inside]
pw = [float(x.split(",")[1]) for x in inside if x.split(",")[1].strip() not in ("[N/A]", "")]
reasons = sorted({x.split(",")[2].strip() for x in inside})
busy = [s for s, p in zip(sm, pw) if p > 400]
print(f"samples {len(sm)}; SM MHz median {statistics.median(sm):.0f} min {min(sm):.0f}; under load (>400 W) "
      f"median {statistics.median(busy) if busy else float('nan'):.0f}; power max {max(pw):.0f} W; reasons {reasons}")
