// Forwarding header: the declarations the reference keeps in hisa/niah.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
