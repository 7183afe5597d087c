OPENQASM 2.0;
include "qelib1.inc";
qreg q[1];
rx(1.5e-1) q[0];
ry(-(pi/2 + 0.25)*2) q[0];
rz(3/4*pi - 1/8) q[0];
u1(0.5*(pi - 1)) q[0];
