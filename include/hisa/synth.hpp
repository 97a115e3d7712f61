// Forwarding header: the declarations the reference keeps in hisa/synth.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
