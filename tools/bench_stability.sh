for i in 1 2 3 4; do
timeout 300 python bench.py --other-configs "" --no-cpu-baseline --no-e2e --no-migration --steps 100 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('q/s %.4e' % d['value'], 'K2 alone %.2f us roofline %.3f' % (d['roofline']['avg_launch_ms'] * 1e3, d['roofline']['frac']), 'eq %.3f' % d['roofline_k2_equal_shares']['frac'], 'K1 %.3f' % d['prefix_roofline']['frac'], 'layers %.3f gaps %.3f' % (b['layers'], b['gaps']))"
done
