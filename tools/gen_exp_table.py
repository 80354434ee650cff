import mpmath, struct
mpmath.mp.prec = 300
N=128
def d2u(x): return struct.unpack('<Q', struct.pack('<d', x))[0]
out=[]
for k in range(N):
    v = mpmath.power(2, mpmath.mpf(k)/N)
    H = float(v)  # mpmath float() rounds to nearest
    T = float((v - mpmath.mpf(H))/mpmath.mpf(H))
    tail = d2u(T)
    sbits = (d2u(H) - ((k << 52)//N)) & ((1<<64)-1)
    out.append((tail, sbits))
print(hex(out[1][0]), hex(out[1][1]), hex(out[2][0]), hex(out[2][1]))
with open('tab.h','w') as f:
    f.write('static const unsigned long long TAB[256]={\n')
    for t,s in out: f.write('0x%016xULL,0x%016xULL,\n'%(t,s))
    f.write('};\n')
