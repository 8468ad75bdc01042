# /proc/stat cpu line (user nice system idle iowait irq softirq steal ...) every 2 s; run in the background
while true; do echo "$(date +%s) $(head -1 /proc/stat)"; sleep 2; done
